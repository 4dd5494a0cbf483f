"""Probe of the host-buffer pipeline: chunk count and H2D stream count vs
the PCIe bound (scripts/pcie.py)."""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2411_09510_b200.collective import HostPipeline  # noqa: E402


def timed(fn, reps=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    n = 2048 * 4096
    h_in = [torch.randn(n).to(torch.bfloat16).pin_memory() for _ in range(2)]
    h_out = torch.empty(n, dtype=torch.bfloat16).pin_memory()
    res = {}
    for hs in (1, 2):
        for k in (2, 4, 8):
            pipe = HostPipeline.simulated("fp4_e2m1:32:e8m0", n, 2, chunks=k, h2d_streams=hs)
            res[f"h2d{hs}_chunks{pipe.k}"] = round(timed(lambda: pipe(h_in, h_out)), 4)
    for w in ((1, 3, 3, 1), (1, 2, 2, 2, 1), (1, 4, 1), (2, 3, 2, 1), (1, 2, 4, 1), (3, 3, 1, 1),
              (1, 6, 1), (2, 5, 1)):
        pipe = HostPipeline.simulated("fp4_e2m1:32:e8m0", n, 2, chunks=w)
        res["pieces" + "-".join(map(str, w))] = round(timed(lambda: pipe(h_in, h_out)), 4)
    pe = HostPipeline.simulated("fp4_e2m1:32:e8m0", n, 2, chunks=4, graph=False)
    res["eager_chunks4"] = round(timed(lambda: pe(h_in, h_out)), 4)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
