"""Prefill TTFT of the TP Llama body: bf16 NCCL all-reduce vs MX-compressed.

    python scripts/ttft.py --model 8b --seq 2048 [--layers L]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/ttft.py --model 70b --seq 4096

One JSON line per (scheme, algo) from rank 0: TTFT ms (max over ranks), and
the speed-up against the bf16 all-reduce.  Random-init weights (std 0.02),
random hidden states; BASELINE.json configs[2] is 70B / seq 4096 / TP=8.
"""

import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2411_09510_b200 import tp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", choices=["8b", "70b"], default="8b")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--seq", type=int, default=2048)
    ap.add_argument("--layers", type=int, default=None, help="truncate the stack (memory)")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--schemes", default="none,fp4_e2m1:32:e8m0")
    ap.add_argument("--graph", action="store_true", help="replay the forward as one CUDA graph")
    ap.add_argument("--algos", default="oneshot,twoshot",
                    help="oneshot,twoshot (NCCL), symm,symm2 (one-kernel NVLink), auto")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = tp.LLAMA31_8B if args.model == "8b" else tp.LLAMA31_70B
    base = None
    for spec in args.schemes.split(","):
        for algo in (["oneshot"] if spec == "none" else args.algos.split(",")):
            scheme = None if spec == "none" else spec
            ms = tp.measure_ttft(cfg, args.batch, args.seq, tp=world, scheme=scheme, algo=algo,
                                 layers=args.layers, reps=args.reps, graph=args.graph)
            if scheme is None:
                base = ms
            if rank == 0:
                print(json.dumps({"model": f"llama-3.1-{args.model}", "tp": world,
                                  "batch": args.batch, "seq": args.seq,
                                  "layers": args.layers or cfg.layers,
                                  "allreduce": "bf16 NCCL" if scheme is None else f"{spec} {algo}",
                                  "ttft_ms": round(ms, 3), "cuda_graph": args.graph,
                                  "speedup_vs_bf16": None if base is None else round(base / ms, 3)}),
                      flush=True)
            torch.cuda.empty_cache()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
