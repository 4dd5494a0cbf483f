"""DRAM traffic of K4 / K1 / K2 over a RANGE of back-to-back launches, write
side included (ncu --replay-mode range; profiles/r02/traffic).

A single-launch ncu capture flushes the caches first and ends with the
kernel's writes still dirty in L2, so it under-counts writes (VERDICT r1,
weak #4).  Here R launches over buffer sets rotated beyond L2 run inside
one cudaProfilerStart/Stop range; the range's dram__bytes_{read,write}
divided by R is the steady-state traffic per launch (at most ~one launch of
writes can still sit in L2 at the end, a <= 1/R error).

    ncu --replay-mode range --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        python scripts/range_traffic.py --kernel k4
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2411_09510_b200.collective import SimulatedAllReduce  # noqa: E402
from paper_2411_09510_b200.formats import parse_scheme  # noqa: E402
from paper_2411_09510_b200.synth import rank_partials  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernel", choices=["k4", "k1", "k2"], default="k4")
    ap.add_argument("--shape", default="2048,4096")
    ap.add_argument("--sets", type=int, default=16)
    ap.add_argument("--scheme", default="fp4_e2m1:32:e8m0")
    args = ap.parse_args()
    T, H = (int(v) for v in args.shape.split(","))
    n = T * H
    sch = parse_scheme(args.scheme, extensions=True)
    dev = torch.device("cuda", 0)
    base = [torch.from_numpy(p).to(dev, torch.bfloat16) for p in rank_partials((T, H), 2, seed=0)]
    sets = [([(b.roll(7 * i, 0) * (-1) ** i).contiguous() for b in base],
             SimulatedAllReduce(sch, n, 2, "oneshot", torch.bfloat16, dev))
            for i in range(args.sets)]
    S = sets[0][1].S

    def launch(i):
        parts, op = sets[i]
        if args.kernel == "k4":
            op(parts)
        elif args.kernel == "k1":
            op.be.quantize_into(parts[0].reshape(-1), op.gathered[0:S], op.ws, op.flag)
        else:
            op.reduce()

    for i in range(args.sets):  # warm: every set touched once, shards valid for k2
        op = sets[i][1]
        op(sets[i][0])
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for i in range(args.sets):
        launch(i)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print(f"kernel={args.kernel} shape={T}x{H} sets={args.sets} shard_bytes={S}")


if __name__ == "__main__":
    main()
