"""Event timeline of one HostPipeline call (eager, timing events between the
stages): when each piece's H2D copies, all-reduce and D2H copy finish,
relative to the call's start.  Diagnoses the gap between the e2e time and
the PCIe bound (scripts/pcie.py)."""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2411_09510_b200.collective import HostPipeline  # noqa: E402


def main():
    n = 2048 * 4096
    h_in = [torch.randn(n).to(torch.bfloat16).pin_memory() for _ in range(2)]
    h_out = torch.empty(n, dtype=torch.bfloat16).pin_memory()
    for k in (2, 4, 8):
        pipe = HostPipeline.simulated("fp4_e2m1:32:e8m0", n, 2, chunks=k, graph=False)
        for _ in range(3):
            pipe(h_in, h_out)
        torch.cuda.synchronize()
        ev = {}
        s_red, s_out, s_in = pipe.streams[0], pipe.streams[1], pipe.streams[2]
        cur = torch.cuda.current_stream()
        t0 = torch.cuda.Event(enable_timing=True)
        t0.record(cur)
        for s in pipe.streams:
            s.wait_stream(cur)
        c = pipe.c
        for j in range(pipe.k):
            sl = slice(j * c, (j + 1) * c)
            with torch.cuda.stream(s_in):
                for d, h in zip(pipe.dev_in, h_in):
                    d[sl].copy_(h[sl], non_blocking=True)
                e = torch.cuda.Event(enable_timing=True)
                e.record(s_in)
                ev[f"h2d{j}"] = e
            with torch.cuda.stream(s_red):
                s_red.wait_event(e)
                pipe.ops[j]([d[sl] for d in pipe.dev_in], pipe.dev_out[sl])
                e2 = torch.cuda.Event(enable_timing=True)
                e2.record(s_red)
                ev[f"red{j}"] = e2
            with torch.cuda.stream(s_out):
                s_out.wait_event(e2)
                h_out[sl].copy_(pipe.dev_out[sl], non_blocking=True)
                e3 = torch.cuda.Event(enable_timing=True)
                e3.record(s_out)
                ev[f"d2h{j}"] = e3
        for s in pipe.streams:
            cur.wait_stream(s)
        torch.cuda.synchronize()
        print(json.dumps({"pieces": k, **{name: round(t0.elapsed_time(e) * 1e3, 1)
                                            for name, e in ev.items()}}))


if __name__ == "__main__":
    main()
