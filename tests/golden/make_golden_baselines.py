"""Golden fixtures for the comparison codecs (TopK, channel-wise INT) made by
running the REAL reference (mx/baselines.py).  Build container only:

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_golden_baselines.py

Writes ``tests/golden/baselines.json``: for every case of ``CASES`` (inputs
regenerated bit-identically by ``tests/golden/inputs.py`` / ``baseline_case``)
the reference's scales (hex f16), SHA-256 of the packed code stream, of the
serialized container and of the float64 decompression (channel INT); the
SHA-256 of the kept indices / f16 values, K and the container digest (TopK).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, "/root/reference/pkg/src")

from mxcomm import baselines as rb  # noqa: E402  (the reference)

from tests.golden.inputs import BASELINE_CASES, baseline_case  # noqa: E402


def sha(b) -> str:
    if isinstance(b, np.ndarray):
        b = np.ascontiguousarray(b).tobytes()
    return hashlib.sha256(b).hexdigest()


def main():
    out = {"chanint": {}, "topk": {}}
    for name in BASELINE_CASES:
        x = baseline_case(name)
        for bits in (2, 3, 4, 5, 8):
            p = rb.channelwise_int_compress(x, bits)
            dec = rb.channelwise_int_decompress(p)
            out["chanint"][f"{name}|{bits}"] = {
                "scales": p.scales.astype("<f2").tobytes().hex() if p.scales.size <= 512
                else sha(p.scales.astype("<f2")),
                "codes": sha(p.code_stream), "code_bytes": len(p.code_stream),
                "container": sha(rb.serialize_channel_int(p)),
                "dec64": sha(dec.astype("<f8")), "nbytes": p.nbytes}
        for factor in (3.0, 4.0, 10.0):
            try:
                p = rb.topk_compress(x, factor)
            except Exception as exc:  # noqa: BLE001
                out["topk"][f"{name}|f{factor:g}"] = {"error": type(exc).__name__}
                continue
            out["topk"][f"{name}|f{factor:g}"] = {
                "k": int(p.k_per_tensor), "indices": sha(p.indices.astype("<u4")),
                "values": sha(p.values.astype("<f2")), "container": sha(rb.serialize_topk(p)),
                "dec64": sha(rb.topk_decompress(p).astype("<f8"))}
        for k in (1, 7, 100):
            p = rb.topk_compress(x, k=k)
            out["topk"][f"{name}|k{k}"] = {
                "k": int(p.k_per_tensor), "indices": sha(p.indices.astype("<u4")),
                "values": sha(p.values.astype("<f2")), "container": sha(rb.serialize_topk(p))}
    # small explicit vectors (hex) for readable failures
    v = np.array([[1.0, -2.0, 0.0, 3.5], [-0.0, 2.0, 0.25, -7.0], [0.5, 0.0, 0.0, 7.0]])
    p = rb.channelwise_int_compress(v, 4)
    out["chanint_vector"] = {"x": v.tolist(), "bits": 4,
                             "scales": p.scales.astype("<f2").tobytes().hex(),
                             "codes": p.code_stream.hex()}
    t = np.array([3.0, -3.0, 1.0, 0.5, -3.0, 2.0, 3.0, 0.0])
    p = rb.topk_compress(t, k=3)
    out["topk_vector"] = {"x": t.tolist(), "k": 3, "indices": p.indices.tolist(),
                          "values": p.values.astype(np.float64).tolist()}
    # simulated TP reports through the baseline codecs (mx/tpsim.py:234-302);
    # the reference's own fp32 partials are stored (BLAS is host-dependent)
    from mxcomm import tpsim as rtp

    out["tpsim"] = []
    for deg, codec_id, seed, ishape, wshape, own in [
            (2, "topk:3", 0, (1, 16, 64), (64, 48), True),
            (4, "chanint:4", 7, (2, 8, 30), (30, 24), True),
            (3, "chanint:8", 3, (1, 8, 25), (25, 16), False),
            (2, "fp16", 1, (1, 16, 64), (64, 64), True),
            (2, "passthrough", 2, (1, 8, 32), (32, 16), True),
            (8, "topk:4", 1, (1, 16, 64), (64, 64), True)]:
        cfg = rtp.TPConfig(deg, codec_id, seed, ishape, wshape, own)
        rep = rtp.simulate_reduction(cfg)
        x, w = rtp.generate_inputs(cfg)
        shards, pad = rtp.shard_rowwise(w, deg)
        if pad:
            x = np.pad(x, [(0, 0)] * (x.ndim - 1) + [(0, pad)])
        rows = shards[0].shape[0]
        parts = [x[..., r * rows:(r + 1) * rows] @ shards[r] for r in range(deg)]
        out["tpsim"].append({"degree": deg, "scheme": codec_id, "seed": seed,
                             "input_shape": ishape, "weight_shape": wshape, "quantize_own": own,
                             "partials_f32_hex": [p.astype(np.float32).tobytes().hex()
                                                  for p in parts],
                             "partial_shape": list(parts[0].shape),
                             "name": rep.scheme,
                             "rel_frob_err": float(rep.rel_frob_err).hex(),
                             "max_abs_err": float(rep.max_abs_err).hex(),
                             "sqnr_db": float(rep.sqnr_db).hex(),
                             "bytes_compressed": rep.bytes_compressed,
                             "bytes_uncompressed": rep.bytes_uncompressed,
                             "padding": rep.padding})
    with open(os.path.join(HERE, "baselines.json"), "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)
    print(f"wrote {len(out['chanint'])} chanint + {len(out['topk'])} topk cases")


if __name__ == "__main__":
    main()
