"""HostPipeline piece layouts / H2D stream counts at the bench workload
(8B partial [2048x4096] bf16, 2 simulated ranks, fp4_e2m1:32:e8m0), one
B200: ms per call (CUDA events, 100 back-to-back calls), plus the PCIe
floors (pinned H2D of both partials, D2H of the result, both concurrently).

    python scripts/e2e_pieces.py
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2411_09510_b200.collective import HostPipeline  # noqa: E402


def timed(fn, reps=100):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps)
    return best


def main():
    n = 2048 * 4096
    dev = torch.device("cuda", 0)
    host_in = [torch.randn(n).to(torch.bfloat16).pin_memory() for _ in range(2)]
    host_out = torch.empty(n, dtype=torch.bfloat16).pin_memory()
    d_in = [torch.empty(n, dtype=torch.bfloat16, device=dev) for _ in range(2)]
    d_out = torch.empty(n, dtype=torch.bfloat16, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def h2d():
        for d, h in zip(d_in, host_in):
            d.copy_(h, non_blocking=True)

    def d2h():
        host_out.copy_(d_out, non_blocking=True)

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            h2d()
        with torch.cuda.stream(s2):
            d2h()
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    print(json.dumps({"floor_h2d_ms": round(timed(h2d), 4), "floor_d2h_ms": round(timed(d2h), 4),
                      "floor_both_ms": round(timed(both), 4)}), flush=True)
    for pieces in ((1, 3, 3, 1), 4, 8, (1, 2, 2, 2, 1), (1, 2, 2, 2, 2, 2, 1), (1, 4, 4, 4, 1),
                   (1, 2, 4, 4, 4, 2, 1), (1, 1, 2, 2, 2, 2, 1, 1), 16):
        for hs in (1, 2):
            pipe = HostPipeline.simulated("fp4_e2m1:32:e8m0", n, 2, "oneshot", torch.bfloat16,
                                          dev, chunks=pieces, h2d_streams=hs)
            ms = timed(lambda: pipe(host_in, host_out))
            print(json.dumps({"pieces": pieces if isinstance(pieces, int) else list(pieces),
                              "h2d_streams": hs, "ms": round(ms, 4),
                              "gbs": round(2 * 2 * n / (ms * 1e-3) / 1e9, 2)}), flush=True)
            del pipe


if __name__ == "__main__":
    main()
