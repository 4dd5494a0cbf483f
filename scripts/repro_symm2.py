"""Repro loop for a fuzz_symm mismatch (K5b two-shot, N concurrent rank
launches on one device): repeat one configuration with fresh random inputs
and report every mismatching (call, rank) with its differing indices, and
whether the wrong values equal a neighbouring call's correct result (stale
slot) or something else.

    python scripts/repro_symm2.py SPEC N n CALLS ITERS [seed]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import mx_oracle as O  # noqa: E402
from paper_2411_09510_b200 import _native  # noqa: E402
from tests.golden import inputs  # noqa: E402
from tests.test_gpu_symm_multirank import run_ranks  # noqa: E402


def main():
    spec, N, n, calls, iters = (sys.argv[1], int(sys.argv[2]), int(sys.argv[3]),
                                int(sys.argv[4]), int(sys.argv[5]))
    algo = sys.argv[7] if len(sys.argv) > 7 else "twoshot"
    rng = np.random.default_rng(int(sys.argv[6]) if len(sys.argv) > 6 else 0)
    f = O.allreduce_oneshot if algo == "oneshot" else O.allreduce_twoshot
    bad, total = [], 0
    for it in range(iters):
        out_dt = torch.float32 if it % 2 == 0 else torch.bfloat16
        x64s, sets = [], []
        for c in range(calls):
            x64 = [inputs.gauss_bf16(n, int(rng.integers(1 << 30))) for _ in range(N)]
            x64s.append(x64)
            sets.append([torch.from_numpy(x).to("cuda", torch.bfloat16) for x in x64])
        outs = run_ranks(_native, spec, sets, calls, out_dtype=out_dt, algo=algo)
        refs = [torch.from_numpy(f(x64s[c], O.scheme(spec))).to(out_dt) for c in range(calls)]
        vt = torch.int16 if out_dt == torch.bfloat16 else torch.int32
        for c, per_rank in enumerate(outs):
            for r, o in enumerate(per_rank):
                total += 1
                a, b = o.cpu().view(vt), refs[c].view(vt)
                if not torch.equal(a, b):
                    idx = (a != b).nonzero().ravel().numpy()
                    stale = [cc for cc in range(calls) if cc != c and
                             torch.equal(a[idx], refs[cc].view(vt)[idx])]
                    bad.append({"iter": it, "call": c, "rank": r, "out": str(out_dt),
                                "ndiff": int(idx.size), "first": int(idx[0]),
                                "last": int(idx[-1]), "chunk_of_first": int(idx[0]) // (n // N),
                                "equals_call": stale,
                                "got0": float(o.cpu()[idx[0]]), "want0": float(refs[c][idx[0]])})
                    print(json.dumps(bad[-1]), flush=True)
    print(json.dumps({"spec": spec, "N": N, "n": n, "calls": calls, "iters": iters,
                      "checked": total, "mismatches": len(bad)}), flush=True)


if __name__ == "__main__":
    main()
