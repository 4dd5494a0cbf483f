"""Achievable-bandwidth reference points at the prefill working-set size.

Times, over buffers rotated through > 3x L2 (cold HBM), graph-captured and
event-timed:
  * torch copy_ of one [2048x4096] bf16 partial (16.8 MB read + 16.8 MB write)
  * torch sum over it (read-only)
  * K1 (mx_quantize) and K2 (mx_dequant_sum, 2 shards) on the same buffers
Prints one JSON line.  Usage: python scripts/membench.py [--shape 2048,4096]
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2411_09510_b200.collective import NativeBackend  # noqa: E402
from paper_2411_09510_b200.formats import parse_scheme  # noqa: E402

L2 = 126 * 2 ** 20


def timed(fn, reps):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(g):
        fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps  # ms per replay


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="2048,4096")
    ap.add_argument("--scheme", default="fp4_e2m1:32:e8m0")
    args = ap.parse_args()
    T, H = map(int, args.shape.split(","))
    n = T * H
    R = max(4, -(-3 * L2 // (2 * n)))
    xs = [torch.randn(n, device="cuda", dtype=torch.bfloat16) for _ in range(R)]
    ys = [torch.empty_like(x) for x in xs]
    sums = torch.empty(R, device="cuda", dtype=torch.bfloat16)
    sch = parse_scheme(args.scheme, extensions=True)
    be = NativeBackend(sch)
    _, _, S = be.layout(n)
    shards = [torch.empty(2 * S, dtype=torch.uint8, device="cuda") for _ in range(R)]
    ws = torch.empty(be.workspace(n), dtype=torch.uint8, device="cuda")
    flag = torch.empty(1, dtype=torch.int64, device="cuda")
    be.reset_flag(flag)
    res = {"n": n, "rotation": R}

    def run(name, body, bytes_per):
        ms = timed(lambda: [body(i) for i in range(R)], 20) / R
        res[name] = {"us": round(ms * 1e3, 3), "GBps": round(bytes_per / ms / 1e6, 1)}

    run("torch_copy", lambda i: ys[i].copy_(xs[i]), 4 * n)
    run("torch_sum", lambda i: torch.sum(xs[i].view(1, -1), dim=1, out=sums[i:i + 1]), 2 * n)
    run("k1_quant", lambda i: be.quantize_into(xs[i], shards[i][:S], ws, flag),
        2 * n + n // 2 + n // 32)
    for i in range(R):
        be.quantize_into(xs[(i + 1) % R], shards[i][S:], ws, flag)
    run("k2_dqsum2", lambda i: be.dequant_sum(shards[i], S, 2, n, n, 0, ys[i]),
        2 * (n // 2 + n // 32) + 2 * n)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
