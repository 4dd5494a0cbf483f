"""Where do HostPipeline's ~0.14 ms over the PCIe floor go?  (probe, not
product.)  Every variant is captured in one CUDA graph and replayed
back-to-back; ms per replay.  Bench workload: two pinned bf16 partials
[2048x4096] in, the pinned bf16 result out.

    python scripts/e2e_gaps.py > gpurun_out/gaps.jsonl
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2411_09510_b200.collective import HostPipeline  # noqa: E402

N = 2048 * 4096


def graph_ms(issue, reps=50):
    issue()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        issue()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps)
    return best


def bounds_of(w):
    units, tot = N // 1024, float(sum(w))
    cuts = [0]
    for x in w[:-1]:
        cuts.append(cuts[-1] + round(units * x / tot))
    cuts.append(units)
    return [c * 1024 for c in cuts]


def main():
    dev = torch.device("cuda", 0)
    hin = [torch.randn(N).to(torch.bfloat16).pin_memory() for _ in range(2)]
    hout = torch.empty(N, dtype=torch.bfloat16).pin_memory()
    din = [torch.empty(N, dtype=torch.bfloat16, device=dev) for _ in range(2)]
    dout = torch.empty(N, dtype=torch.bfloat16, device=dev)
    hcat = torch.empty(2 * N, dtype=torch.bfloat16).pin_memory()
    dcat = torch.empty(2 * N, dtype=torch.bfloat16, device=dev)
    sA, sB, sC = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    rows = []

    def rec(name, fn, **kw):
        r = {"what": name, "ms": round(graph_ms(fn), 4), **kw}
        rows.append(r)
        print(json.dumps(r), flush=True)

    def fork(*ss):
        cur = torch.cuda.current_stream()
        for s in ss:
            s.wait_stream(cur)

    def join(*ss):
        cur = torch.cuda.current_stream()
        for s in ss:
            cur.wait_stream(s)

    rec("H2D 2 whole copies", lambda: [d.copy_(h, non_blocking=True) for d, h in zip(din, hin)])
    rec("H2D 1 copy of 2n (contiguous host)", lambda: dcat.copy_(hcat, non_blocking=True))
    rec("D2H whole", lambda: hout.copy_(dout, non_blocking=True))

    def both():
        fork(sA, sB)
        with torch.cuda.stream(sA):
            for d, h in zip(din, hin):
                d.copy_(h, non_blocking=True)
        with torch.cuda.stream(sB):
            hout.copy_(dout, non_blocking=True)
        join(sA, sB)

    rec("H2D + D2H concurrent (floor)", both)
    layouts = ((1, 3, 3, 1), (1, 1, 1, 1), (1, 2, 2, 2, 2, 1))
    if len(sys.argv) > 1:  # tail-decreasing sweep: HostPipeline only
        for spec in sys.argv[1:]:
            w = tuple(int(v) for v in spec.split(","))
            pipe = HostPipeline.simulated("fp4_e2m1:32:e8m0", N, 2, chunks=w, graph=False)
            rec(f"HostPipeline {w}", lambda: pipe._issue(hin, hout))
            del pipe
        return
    for w in layouts:
        b = bounds_of(w)

        def h2d_pieces(b=b):
            for j in range(len(b) - 1):
                sl = slice(b[j], b[j + 1])
                for d, h in zip(din, hin):
                    d[sl].copy_(h[sl], non_blocking=True)

        rec(f"H2D pieces {w}", h2d_pieces)

        def copies_pipe(b=b):
            fork(sA, sB)
            for j in range(len(b) - 1):
                sl = slice(b[j], b[j + 1])
                with torch.cuda.stream(sA):
                    for d, h in zip(din, hin):
                        d[sl].copy_(h[sl], non_blocking=True)
                    e = torch.cuda.Event()
                    e.record(sA)
                with torch.cuda.stream(sB):
                    sB.wait_event(e)
                    hout[sl].copy_(dout[sl], non_blocking=True)
            join(sA, sB)

        rec(f"copies-only pipeline {w}", copies_pipe)
        pipe = HostPipeline.simulated("fp4_e2m1:32:e8m0", N, 2, chunks=w, graph=False)
        rec(f"HostPipeline {w}", lambda: pipe._issue(hin, hout))
        pipe2 = HostPipeline.simulated("fp4_e2m1:32:e8m0", N, 2, chunks=w, graph=False,
                                       h2d_streams=2)
        rec(f"HostPipeline {w} 2 H2D streams", lambda: pipe2._issue(hin, hout))
        del pipe, pipe2


if __name__ == "__main__":
    main()
