"""Randomised multi-rank sweep of the NVLink kernels (K5 one-shot, K5b
two-shot) on one device: N concurrent rank launches over peer pointers
(tests/test_gpu_symm_multirank.py), random schemes / sizes / N / output
dtypes, several consecutive calls per configuration; bit-exact against the
oracle on every rank.

    python scripts/fuzz_symm.py [seconds] [seed]
"""

import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import mx_oracle as O  # noqa: E402
from paper_2411_09510_b200 import _native  # noqa: E402
from tests.golden import inputs  # noqa: E402
from tests.test_gpu_symm_multirank import run_ranks  # noqa: E402

SPECS = [f"{e}:{b}:e8m0" for e in ("fp4_e2m1", "fp6_e2m3", "fp6_e3m2", "int8", "fp5_e2m2")
         for b in (16, 32, 64)]


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 60.0
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    t0, cases, fails = time.time(), 0, []
    while time.time() - t0 < budget:
        spec = SPECS[rng.integers(len(SPECS))]
        N = int(rng.integers(1, 9))
        algo = "oneshot" if rng.random() < 0.5 else "twoshot"
        units = int(rng.integers(1, 9)) * (N if algo == "twoshot" else 1)
        n = units * 1024  # <= 64 units per rank: every rank's CTAs co-resident
        out_dt = torch.float32 if rng.random() < 0.5 else torch.bfloat16
        calls = int(rng.integers(1, 4))
        sets, x64s = [], []
        for c in range(calls):
            x64 = [inputs.gauss_bf16(n, int(rng.integers(1 << 30))) for _ in range(N)]
            x64s.append(x64)
            sets.append([torch.from_numpy(x).to("cuda", torch.bfloat16) for x in x64])
        try:
            outs = run_ranks(_native, spec, sets, calls, out_dtype=out_dt, algo=algo)
            ok = True
            for c, per_rank in enumerate(outs):
                f = O.allreduce_oneshot if algo == "oneshot" else O.allreduce_twoshot
                ref = torch.from_numpy(f(x64s[c], O.scheme(spec))).to(out_dt)
                for o in per_rank:
                    a = o.cpu().view(torch.int16 if out_dt == torch.bfloat16 else torch.int32)
                    b = ref.view(torch.int16 if out_dt == torch.bfloat16 else torch.int32)
                    ok = ok and torch.equal(a, b)
        except Exception as exc:  # noqa: BLE001
            ok = False
            spec += f" EXC {type(exc).__name__}: {exc}"[:200]
        cases += 1
        if not ok:
            fails.append({"spec": spec, "N": N, "n": n, "algo": algo, "calls": calls})
    print(json.dumps({"cases": cases, "failures": len(fails), "first": fails[:10],
                      "seconds": round(time.time() - t0, 1)}))
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
