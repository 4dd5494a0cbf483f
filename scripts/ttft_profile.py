"""Per-kernel device time of the TTFT forward replayed as a CUDA graph
(torch.profiler / CUPTI kernel records; no replay serialisation, unlike
ncu): which kernels make the MX path slower or faster than bf16.

    python scripts/ttft_profile.py --layers 8 [--scheme fp4_e2m1:32:e8m0]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2411_09510_b200 import tp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--seq", type=int, default=2048)
    ap.add_argument("--scheme", default="none")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    scheme = None if args.scheme == "none" else args.scheme
    _, _, _, LlamaTP = tp.make_module_classes()
    torch.manual_seed(0)
    model = LlamaTP(tp.LLAMA31_8B, 1, None, scheme, "oneshot", args.layers)
    h = torch.randn(1, args.seq, tp.LLAMA31_8B.hidden, device="cuda", dtype=torch.bfloat16)
    with torch.inference_mode():
        for _ in range(2):
            model(h)
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            model(h)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            model(h)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        from torch.profiler import ProfilerActivity, profile

        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(args.reps):
                g.replay()
            torch.cuda.synchronize()
    rows = []
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    agg = {}
    t0, t1 = None, None
    for e in evs:
        name = e.name.split("(")[0][:90]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += e.device_time_range.elapsed_us() if hasattr(e, "device_time_range") else (
            e.time_range.elapsed_us())
        st, en = e.time_range.start, e.time_range.end
        t0 = st if t0 is None else min(t0, st)
        t1 = en if t1 is None else max(t1, en)
    tot = sum(v[1] for v in agg.values())
    for name, (cnt, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        rows.append({"kernel": name, "launches": cnt // args.reps,
                     "us_per_forward": round(us / args.reps, 1)})
    for r in rows:
        print(json.dumps(r))
    print(json.dumps({"scheme": args.scheme, "layers": args.layers,
                      "kernel_us_per_forward": round(tot / args.reps, 1),
                      "span_us_per_forward": round((t1 - t0) / args.reps, 1) if t0 else None}))


if __name__ == "__main__":
    main()
