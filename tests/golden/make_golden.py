"""Generate the golden parity fixtures by running the REAL reference.

Run in the build container only (the reference is not shipped to the GPU
box):

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_golden.py

Writes ``tests/golden/golden.json``:

* ``vectors``  -- small hand-picked inputs with full hex streams (SPEC.md
  worked examples: SPEC.md:130-132, 148; SURVEY.md §8(c) extras);
* ``digests``  -- SHA-256 of scale stream / element stream / float32 and
  float64 decompression for every (case, scheme) of ``inputs.CASES`` x
  ``inputs.sweep_schemes()``;
* ``decode``   -- SHA-256 of the reference's decompression of random byte
  streams (every code point, every scale code incl. 2^128 -> inf);
* ``reduce``   -- SHA-256 of the netbench fp32 rank-order sum
  (mx/netbench.py:332-334) over 3 ranks for a few schemes;
* ``large``    -- SHA-256 of the streams for the 8B prefill shape
  [2048x4096] (gaussian_with_outliers seed 0, bf16) and of the TP=2 one-shot
  reduction (seeds 0,1), per BASELINE.json sweep scheme;
* ``nonfinite`` -- block index reported for NaN/Inf inputs.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, "/root/reference/pkg/src")

import mxcomm  # noqa: E402  (the reference)
from mxcomm import codec as rcodec  # noqa: E402
from mxcomm import formats as rformats  # noqa: E402
from mxcomm import netbench as rnet  # noqa: E402
from mxcomm import synth as rsynth  # noqa: E402

from tests.golden import inputs  # noqa: E402
from paper_2411_09510_b200 import synth as mysynth  # noqa: E402

EXT = {
    "fp6_e2m3": (rformats.FormatKind.FLOAT_MICRO, 2, 3),
    "fp6_e3m2": (rformats.FormatKind.FLOAT_MICRO, 3, 2),
    "int8": (rformats.FormatKind.INT_SYMMETRIC, 0, 7),
    "fp3_e2m0": (rformats.FormatKind.FLOAT_MICRO, 2, 0),
    "fp8_e4m3": (rformats.FormatKind.FLOAT_MICRO, 4, 3),
    "fp8_e5m2": (rformats.FormatKind.FLOAT_MICRO, 5, 2),
}


def ref_scheme(spec: str):
    el, blk, sc = spec.split(":")
    if el in rformats.ELEMENT_FORMATS:
        elem = rformats.ELEMENT_FORMATS[el]
    else:
        k, e, m = EXT[el]
        elem = rformats.ElementFormat(k, e, m)
    return rformats.SchemeDescriptor(elem, int(blk), rformats.SCALE_FORMATS[sc])


def sha(b) -> str:
    if isinstance(b, np.ndarray):
        b = np.ascontiguousarray(b).tobytes()
    return hashlib.sha256(b).hexdigest()


def main():
    t0 = time.time()
    out = {"generator": "tests/golden/make_golden.py", "reference": "mxcomm "
           + mxcomm.__version__, "vectors": [], "digests": {}, "decode": {},
           "reduce": {}, "large": {}, "nonfinite": []}

    # -- synth restatement must reproduce the reference generator ---------
    for shape, seed in [((4099,), 3), ((64, 33), 11)]:
        a = rsynth.gaussian_with_outliers(np.random.default_rng(seed), shape)
        b = mysynth.gaussian_with_outliers(np.random.default_rng(seed), shape)
        assert a.tobytes() == b.tobytes(), "synth restatement diverged"

    # -- explicit vectors --------------------------------------------------
    vecs = [
        ("spec_130", [1.0, -6.0, 0.25, 3.0], "fp4_e2m1:32:e8m0"),
        ("spec_131_zero", [0.0, 0.0, -0.0, 0.0], "fp4_e2m1:32:e8m0"),
        ("spec_132_clamp", [2.0 ** 130, 1.0], "fp4_e2m1:32:e5m0"),
        ("overshoot", [7.0, 1.0], "fp4_e2m1:32:e8m0"),
        ("signed_zero", [-0.1, 6.0, -0.0, 0.0], "fp4_e2m1:32:e8m0"),
        ("n70", list(np.linspace(-3, 5, 70)), "fp4_e2m1:32:e8m0"),
        ("e5m0_ones_9blocks", [1.0] * (9 * 32), "fp4_e2m1:32:e5m0"),
        ("fp5_e2m2_b8", [1, 2, 3, 4, 5, 6, 7, 0.25], "fp5_e2m2:8:e8m0"),
        ("int4_ties", [0.5, 1.5, 2.5, -3.5, 7.0, 7.5, -0.49, 6.5], "int4:8:e8m0"),
        ("fp2_ties", [1.0, 0.5, 1.5, -2.0, 3.0, 0.0, -1.0, 2.0], "fp2_e1m0:8:e8m0"),
        ("e2m0_ties", [3.0, 1.5, 0.5, 6.0, 0.75, 2.0, -3.0, 1.0], "fp3_e2m0:8:e8m0"),
        ("tiny_subnormal_block", [1e-45, -1e-45, 2e-45, 0.0], "fp4_e2m1:4:e8m0"),
        ("huge_block", [3.4e38, -1e38, 1.0, -2.0], "fp4_e2m1:4:e8m0"),
        ("int8_b64", list(np.linspace(-100, 27.3, 64)), "int8:64:e8m0"),
        ("fp6_b16", list(np.linspace(-7.1, 19.9, 37)), "fp6_e2m3:16:e8m0"),
    ]
    for name, vals, spec in vecs:
        sch = ref_scheme(spec)
        arr = np.asarray(vals, dtype=np.float64)
        ct = rcodec.compress_tensor(arr, sch)
        dec = rcodec.decompress_tensor(ct, dtype=np.float64)
        out["vectors"].append({
            "name": name, "scheme": spec, "values": [float(v) for v in arr],
            "values_hex": [float(v).hex() for v in arr],
            "scale_stream": ct.scale_stream.hex(),
            "element_stream": ct.element_stream.hex(),
            "decoded_hex": [float(v).hex() for v in dec],
        })

    # -- digests over the sweep -------------------------------------------
    schemes = inputs.sweep_schemes()
    for cname, (gen, dtype) in inputs.CASES.items():
        x = gen()
        out["digests"][cname] = {"dtype": dtype, "n": int(x.size),
                                 "input_sha": sha(x.astype(np.float64)), "schemes": {}}
        for spec in schemes:
            sch = ref_scheme(spec)
            ct = rcodec.compress_tensor(x, sch)
            d32 = rcodec.decompress_tensor(ct, dtype=np.float32)
            d64 = rcodec.decompress_tensor(ct, dtype=np.float64)
            out["digests"][cname]["schemes"][spec] = {
                "scale": sha(ct.scale_stream), "elem": sha(ct.element_stream),
                "dec32": sha(d32), "dec64": sha(d64),
                "nbytes": [len(ct.scale_stream), len(ct.element_stream)],
            }
        print(f"[golden] {cname}: {len(schemes)} schemes  t={time.time()-t0:.1f}s", flush=True)

    # -- decode of random streams ------------------------------------------
    for spec in schemes:
        sch = ref_scheme(spec)
        n = 4099
        nb = -(-n // sch.block_size)
        ss, es = inputs.random_streams(
            mxcomm.bitpack.packed_nbytes(nb, sch.scale.exponent_bits),
            mxcomm.bitpack.packed_nbytes(n, sch.element.total_bits), seed=sum(map(ord, spec)))
        ct = rcodec.CompressedTensor(sch, (n,), ss, es)
        with np.errstate(over="ignore"):
            d32 = rcodec.decompress_tensor(ct, dtype=np.float32)
        d64 = rcodec.decompress_tensor(ct, dtype=np.float64)
        out["decode"][spec] = {"n": n, "seed": sum(map(ord, spec)),
                               "dec32": sha(d32), "dec64": sha(d64)}

    # -- netbench rank-order reduction --------------------------------------
    for spec in ["fp4_e2m1:32:e8m0", "fp5_e2m2:16:e8m0", "int8:32:e8m0",
                 "fp6_e3m2:64:e8m0", "fp4_e2m1:7:e5m0"]:
        sch = ref_scheme(spec)
        parts = [inputs.gauss_bf16(4099, 100 + r) for r in range(3)]
        acc = np.zeros(4099, dtype=np.float32)
        for p in parts:  # fixed rank order, +0.0 init (mx/netbench.py:332-334)
            if spec.split(":")[0] in rformats.ELEMENT_FORMATS:
                own = rnet._BlockWire(sch, (4099,)).encode_with_reconstruction(p)[1]
            else:  # _BlockWire.serialize rejects non-registry formats (mx/codec.py:337)
                own = rcodec.decompress_tensor(rcodec.compress_tensor(p, sch), dtype=np.float32)
            acc += own
        out["reduce"][spec] = {"ranks": 3, "n": 4099, "seeds": [100, 101, 102],
                               "sum32": sha(acc)}

    # -- non-finite ----------------------------------------------------------
    for idx, bad, blk in [(40, np.nan, 32), (0, np.inf, 32), (100, -np.inf, 7), (4000, np.nan, 64)]:
        x = np.ones(4099)
        x[idx] = bad
        x[4098] = np.nan  # a later one must not win
        try:
            rcodec.compress_tensor(x, ref_scheme(f"fp4_e2m1:{blk}:e8m0"))
            got = None
        except mxcomm.errors.NonFiniteInput as e:
            got = e.block_index
        out["nonfinite"].append({"index": idx, "value": str(bad), "block": blk, "block_index": got})

    # -- simulated TP reduction reports (mx/tpsim.py:234-302) ------------------
    from mxcomm import tpsim as rtp
    out["tpsim"] = []
    for deg, spec, seed, ishape, wshape, own in [
            (2, "fp4_e2m1:32:e8m0", 0, (1, 16, 64), (64, 48), True),
            (4, "fp5_e2m2:16:e5m0", 7, (2, 8, 30), (30, 24), True),
            (3, "int4:8:e8m0", 3, (1, 8, 25), (25, 16), False),
            (8, "fp4_e2m1:32:e8m0", 1, (1, 16, 64), (64, 64), True)]:
        cfg = rtp.TPConfig(deg, rformats.parse_scheme(spec), seed, ishape, wshape, own)
        rep = rtp.simulate_reduction(cfg)
        # the reference's own fp32 partials (BLAS results depend on the host
        # CPU, so they are stored; mx/tpsim.py:251-263)
        x, w = rtp.generate_inputs(cfg)
        shards, pad = rtp.shard_rowwise(w, deg)
        if pad:
            x = np.pad(x, [(0, 0)] * (x.ndim - 1) + [(0, pad)])
        rows = shards[0].shape[0]
        parts = [x[..., r * rows:(r + 1) * rows] @ shards[r] for r in range(deg)]
        out["tpsim"].append({"degree": deg, "scheme": spec, "seed": seed, "input_shape": ishape,
                             "weight_shape": wshape, "quantize_own": own,
                             "partials_f32_hex": [p.astype(np.float32).tobytes().hex()
                                                  for p in parts],
                             "partial_shape": list(parts[0].shape),
                             "rel_frob_err": float(rep.rel_frob_err).hex(),
                             "max_abs_err": float(rep.max_abs_err).hex(),
                             "sqnr_db": float(rep.sqnr_db).hex(),
                             "bytes_compressed": rep.bytes_compressed,
                             "bytes_uncompressed": rep.bytes_uncompressed, "padding": rep.padding})

    # -- large prefill shape -------------------------------------------------
    T, H = inputs.LARGE_SHAPE
    p0 = mysynth.bf16_round(rsynth.gaussian_with_outliers(np.random.default_rng(0), (T, H)))
    p1 = mysynth.bf16_round(rsynth.gaussian_with_outliers(np.random.default_rng(1), (T, H)))
    out["large"]["shape"] = [T, H]
    out["large"]["input_sha"] = [sha(p0), sha(p1)]
    for spec in inputs.LARGE_SCHEMES:
        sch = ref_scheme(spec)
        ct0 = rcodec.compress_tensor(p0, sch)
        ct1 = rcodec.compress_tensor(p1, sch)
        acc = np.zeros((T, H), dtype=np.float32)
        acc += rcodec.decompress_tensor(ct0, dtype=np.float32)
        acc += rcodec.decompress_tensor(ct1, dtype=np.float32)
        out["large"][spec] = {"scale": sha(ct0.scale_stream), "elem": sha(ct0.element_stream),
                              "nbytes": [len(ct0.scale_stream), len(ct0.element_stream)],
                              "tp2_sum32": sha(acc)}
        print(f"[golden] large {spec} t={time.time()-t0:.1f}s", flush=True)

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)
    print(f"[golden] wrote golden.json in {time.time()-t0:.1f}s")


if __name__ == "__main__":
    main()
