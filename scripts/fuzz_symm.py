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
    """argv: seconds seed [first_case last_case]: with a case range, the
    generator is fast-forwarded (no GPU work) and only those cases run --
    the replay of a reported failure ("case" in its record)."""
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 60.0
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    lo = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    hi = int(sys.argv[4]) if len(sys.argv) > 4 else None
    t0, cases, fails, case = time.time(), 0, [], -1
    while time.time() - t0 < budget:
        case += 1
        if hi is not None and case > hi:
            break
        spec = SPECS[rng.integers(len(SPECS))]
        N = int(rng.integers(1, 9))
        algo = "oneshot" if rng.random() < 0.5 else "twoshot"
        algo = os.environ.get("FUZZ_ALGO", algo)
        units = int(rng.integers(1, 9)) * (N if algo == "twoshot" else 1)
        n = units * 1024  # <= 64 units per rank: every rank's CTAs co-resident
        out_dt = torch.float32 if rng.random() < 0.5 else torch.bfloat16
        calls = int(rng.integers(1, 4))
        seeds = [[int(rng.integers(1 << 30)) for _ in range(N)] for _ in range(calls)]
        if case < lo:
            continue
        sets, x64s = [], []
        for c in range(calls):
            x64 = [inputs.gauss_bf16(n, sd) for sd in seeds[c]]
            x64s.append(x64)
            sets.append([torch.from_numpy(x).to("cuda", torch.bfloat16) for x in x64])
        try:
            outs = run_ranks(_native, spec, sets, calls, out_dtype=out_dt, algo=algo)
            ok = True
            f = O.allreduce_oneshot if algo == "oneshot" else O.allreduce_twoshot
            vt = torch.int16 if out_dt == torch.bfloat16 else torch.int32
            refs = [torch.from_numpy(f(x64s[c], O.scheme(spec))).to(out_dt).view(vt)
                    for c in range(calls)]
            detail = []
            for c, per_rank in enumerate(outs):
                for r, o in enumerate(per_rank):
                    a = o.cpu().view(vt)
                    if not torch.equal(a, refs[c]):
                        ok = False
                        idx = (a != refs[c]).nonzero().ravel().numpy()
                        detail.append({"call": c, "rank": r, "ndiff": int(idx.size),
                                       "first": int(idx[0]), "last": int(idx[-1]),
                                       "chunk": int(idx[0]) // max(1, n // N),
                                       "equals_call": [cc for cc in range(calls) if cc != c and
                                                       torch.equal(a[idx], refs[cc][idx])],
                                       "zero": bool((a[idx] == 0).all())})
        except Exception as exc:  # noqa: BLE001
            ok, detail = False, None
            spec += f" EXC {type(exc).__name__}: {exc}"[:200]
        cases += 1
        if not ok:
            fails.append({"case": case, "spec": spec, "N": N, "n": n, "algo": algo,
                          "calls": calls, "out": str(out_dt),
                          "detail": detail[:8] if "EXC" not in spec else None})
            print(json.dumps(fails[-1]), flush=True)
    print(json.dumps({"cases": cases, "failures": len(fails), "first": fails[:10],
                      "seconds": round(time.time() - t0, 1)}))
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
