"""Pin the comparison-codec oracle (TopK, channel-wise INT) against the
reference's own outputs (tests/golden/baselines.json, made by
tests/golden/make_golden_baselines.py from mx/baselines.py)."""

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import baselines_oracle as BO
from tests.golden import inputs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def sha(b):
    if isinstance(b, np.ndarray):
        b = np.ascontiguousarray(b).tobytes()
    return hashlib.sha256(b).hexdigest()


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(ROOT, "tests", "golden", "baselines.json")) as f:
        return json.load(f)


SMALL = [c for c in inputs.BASELINE_CASES if not c.startswith("prefill")]


@pytest.mark.parametrize("case", SMALL)
@pytest.mark.parametrize("bits", [2, 3, 4, 5, 8])
def test_chanint_matches_reference(gold, case, bits):
    g = gold["chanint"][f"{case}|{bits}"]
    x = inputs.baseline_case(case)
    s16, codes, stream = BO.chanint_compress(x, bits)
    sb = s16.astype("<f2").tobytes()
    assert g["scales"] in (sb.hex(), sha(sb))
    assert sha(stream) == g["codes"] and len(stream) == g["code_bytes"]
    dec = BO.chanint_decompress(s16, stream, x.shape, bits)
    assert sha(dec.astype("<f8")) == g["dec64"]


@pytest.mark.parametrize("case", SMALL)
def test_topk_matches_reference(gold, case):
    x = inputs.baseline_case(case)
    for key, g in gold["topk"].items():
        name, arg = key.split("|")
        if name != case or "error" in g:
            continue
        if arg.startswith("f"):
            idx, vals = BO.topk_compress(x, factor=float(arg[1:]))
        else:
            idx, vals = BO.topk_compress(x, k=int(arg[1:]))
        assert idx.size == g["k"], key
        assert sha(idx.astype("<u4")) == g["indices"], key
        assert sha(vals.astype("<f2")) == g["values"], key
        if "dec64" in g:
            assert sha(BO.topk_decompress(idx, vals, x.shape).astype("<f8")) == g["dec64"], key


def test_explicit_vectors(gold):
    v = gold["chanint_vector"]
    s16, codes, stream = BO.chanint_compress(np.array(v["x"]), v["bits"])
    assert s16.astype("<f2").tobytes().hex() == v["scales"] and stream.hex() == v["codes"]
    t = gold["topk_vector"]
    idx, vals = BO.topk_compress(np.array(t["x"]), k=t["k"])
    assert idx.tolist() == t["indices"] and vals.astype(np.float64).tolist() == t["values"]


@pytest.mark.slow
def test_prefill_shape(gold):
    x = inputs.baseline_case("prefill_bf16_2048x4096")
    s16, _, stream = BO.chanint_compress(x, 4)
    g = gold["chanint"]["prefill_bf16_2048x4096|4"]
    assert sha(s16.astype("<f2")) == g["scales"] and sha(stream) == g["codes"]
    idx, vals = BO.topk_compress(x, factor=3.0)
    g = gold["topk"]["prefill_bf16_2048x4096|f3"]
    assert sha(idx.astype("<u4")) == g["indices"] and sha(vals.astype("<f2")) == g["values"]
