"""Randomised parity sweep (GPU vs the pinned oracle), beyond the fixed
cases of tests/: random schemes, sizes (including non-multiples of the
block and of 1024), rank counts, algorithms, output dtypes and input
distributions.  Every result must be bit-identical.

    python scripts/fuzz_parity.py [seconds] [seed]
"""

import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import mx_oracle as O  # noqa: E402
from oracle import baselines_oracle as BO  # noqa: E402
from paper_2411_09510_b200 import baselines as BL  # noqa: E402
from paper_2411_09510_b200 import (compress_tensor_device, decompress_tensor_device,  # noqa: E402
                                   parse_scheme)
from paper_2411_09510_b200.collective import SimulatedAllReduce  # noqa: E402
from paper_2411_09510_b200.synth import bf16_round  # noqa: E402

ELEMS = ["fp4_e2m1", "fp5_e2m2", "fp5_e3m1", "fp5_e1m3", "fp4_e1m2", "fp3_e1m1", "fp2_e1m0",
         "int3", "int4", "int5", "fp6_e2m3", "fp6_e3m2", "int8", "fp3_e2m0", "fp8_e4m3",
         "fp8_e5m2"]
BLOCKS = [8, 16, 32, 64, 7, 24, 100]
SCALES = ["e8m0", "e5m0", "e4m0", "e6m0", "e7m0"]


def sample(rng, n, kind=None):
    kind = rng.integers(0, 4) if kind is None else kind
    if kind == 0:
        x = rng.standard_normal(n)
        x[rng.random(n) < 0.01] *= 100
    elif kind == 1:
        x = rng.standard_normal(n) * 10.0 ** rng.uniform(-30, 30)
    elif kind == 2:
        x = np.where(rng.random(n) < 0.3, 0.0, rng.standard_normal(n))
        x[rng.random(n) < 0.05] = -0.0
    else:
        x = rng.choice(np.array([0.5, 1.0, 1.5, 3.0, 6.0, -4.0, 0.25]), size=n) * 2.0 ** rng.integers(-8, 8)
    return bf16_round(x.astype(np.float32)).astype(np.float64)


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    t0, cases, fails = time.time(), 0, []
    while time.time() - t0 < budget:
        el = ELEMS[rng.integers(len(ELEMS))]
        blk = int(BLOCKS[rng.integers(len(BLOCKS))])
        sc = SCALES[rng.integers(len(SCALES))] if rng.random() < 0.3 else "e8m0"
        spec = f"{el}:{blk}:{sc}"
        n = int(rng.choice([rng.integers(1, 5000), 1024 * int(rng.integers(1, 64)),
                            int(rng.integers(1, 300)) * 1024 + int(rng.integers(0, 1024))]))
        N = int(rng.integers(1, 9))
        algo = "twoshot" if (N > 1 and rng.random() < 0.4) else "oneshot"
        out_dt = torch.float32 if rng.random() < 0.5 else torch.bfloat16
        kind = int(rng.integers(0, 4))
        x64 = [sample(rng, n, kind) for _ in range(N)]
        parts = [torch.from_numpy(x).to("cuda", torch.bfloat16) for x in x64]
        osch = O.scheme(spec)
        try:
            # codec streams of rank 0, fed as bf16 / f16 / f32 (values are
            # bf16-exact, so all three must give the same streams)
            in_dt = [torch.bfloat16, torch.float16, torch.float32][int(rng.integers(0, 3))]
            xin = torch.from_numpy(x64[0]).to("cuda", in_dt)
            x0 = xin.double().cpu().numpy()  # f16 may round/overflow: the fed values
            d = compress_tensor_device(xin, parse_scheme(spec, extensions=True),
                                       check_finite=False)
            ss, es = O.compress(x0, osch) if np.isfinite(x0).all() else (None, None)
            ok = ss is None or (d.scale.cpu().numpy().tobytes() == ss and
                                d.elements.cpu().numpy().tobytes() == es)
            stage = "codec" if not ok else None
            if ok and ss is not None:  # plain decode (decompress_tensor) to f32
                dec = decompress_tensor_device(d, torch.float32).cpu().numpy().ravel()
                ref_dec = O.decompress(ss, es, n, osch, np.float32)
                if not np.array_equal(dec.view(np.uint32), np.asarray(ref_dec, np.float32).view(np.uint32)):
                    ok, stage = False, "decompress"
            # the all-reduce (fused where eligible)
            op = SimulatedAllReduce(spec, n, N, algo, out_dt)
            got = op(parts).float().cpu().numpy()
            ref = (O.allreduce_oneshot if algo == "oneshot" else O.allreduce_twoshot)(x64, osch)
            want = torch.from_numpy(ref).to(out_dt).float().numpy()
            same = got.view(np.uint32) == want.view(np.uint32)
            if ok and not same.all():
                stage = "reduce"
                bad = int(np.flatnonzero(~same)[0])
                stage += f" i={bad} got={got[bad]!r} want={want[bad]!r} nbad={int((~same).sum())}"
                ok = False
        except Exception as exc:  # noqa: BLE001
            ok = False
            spec += f" EXC {type(exc).__name__}: {exc}"[:200]
        # comparison codecs on a 2-D view of rank 0's partial
        if ok and rng.random() < 0.3:
            try:
                C = min(n, int(rng.choice([8, 16, 24, 40, 64, 128, 1000])))
                rows = max(1, n // C)
                xm = x64[0][: rows * C].reshape(rows, C)
                dt = [torch.bfloat16, torch.float32][int(rng.integers(0, 2))]
                xt = torch.from_numpy(xm).to("cuda", dt)
                xv = xt.double().cpu().numpy()
                bits = int(rng.integers(2, 9))
                p = BL.channelwise_int_compress(xt, bits)
                s16, _, stream = BO.chanint_compress(xv, bits)
                k = int(rng.integers(1, xv.size + 1))
                q = BL.topk_compress(xt, k=k)
                ri, rv = BO.topk_compress(xv, k=k)
                if not (p.code_stream == stream and np.array_equal(p.scales.view(np.uint16), s16.view(np.uint16))):
                    ok, stage = False, f"chanint bits={bits} C={C}"
                elif not (np.array_equal(q.indices, ri) and np.array_equal(q.values.view(np.uint16), rv.view(np.uint16))):
                    ok, stage = False, f"topk k={k}"
            except Exception as exc:  # noqa: BLE001
                ok, stage = False, f"baselines EXC {type(exc).__name__}: {exc}"[:200]
        cases += 1
        if not ok:
            fails.append({"spec": spec, "n": n, "N": N, "algo": algo, "out": str(out_dt),
                          "kind": kind, "stage": locals().get("stage")})
    from collections import Counter
    by = Counter((f["kind"], f["algo"], (f["stage"] or "exc")[:6]) for f in fails)
    print(json.dumps({"by_kind_algo_stage": {str(k): v for k, v in by.items()}}))
    print(json.dumps({"cases": cases, "failures": len(fails), "first": fails[:10],
                      "seconds": round(time.time() - t0, 1)}))
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
