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


@pytest.mark.parametrize("case", SMALL)
def test_host_containers_match_reference(gold, case):
    """The product package's MXC1 container formatting for the comparison
    codecs (host code, no GPU) reproduces the reference's bytes."""
    from paper_2411_09510_b200 import baselines as bl

    x = inputs.baseline_case(case)
    for bits in (2, 4, 8):
        s16, _, stream = BO.chanint_compress(x, bits)
        p = bl.ChannelIntPacket(shape=tuple(x.shape) or (1,), bits=bits, scales=s16,
                                code_stream=stream)
        blob = bl.serialize_channel_int(p)
        assert sha(blob) == gold["chanint"][f"{case}|{bits}"]["container"]
        q = bl.deserialize_channel_int(blob)
        assert q.code_stream == stream and np.array_equal(q.scales, s16) and q.bits == bits
        assert p.nbytes == gold["chanint"][f"{case}|{bits}"]["nbytes"]
    for key, g in gold["topk"].items():
        name, arg = key.split("|")
        if name != case or "error" in g:
            continue
        if arg.startswith("f"):
            k = bl.topk_budget(x.size, x.ndim, float(arg[1:]))
        else:
            k = int(arg[1:])
        idx, vals = BO.topk_compress(x, k=k)
        p = bl.TopKPacket(shape=tuple(x.shape), indices=idx, values=vals)
        blob = bl.serialize_topk(p)
        assert sha(blob) == g["container"], key
        q = bl.deserialize_topk(blob)
        assert np.array_equal(q.indices, idx) and np.array_equal(q.values.view(np.uint16),
                                                               vals.view(np.uint16))


def test_host_container_errors():
    from paper_2411_09510_b200 import baselines as bl
    from paper_2411_09510_b200.errors import MalformedHeader, TruncatedStream

    p = bl.TopKPacket(shape=(4, 4), indices=np.array([1, 5], np.uint32),
                      values=np.array([1.0, -2.0], np.float16))
    blob = bl.serialize_topk(p)
    with pytest.raises(TruncatedStream):
        bl.deserialize_topk(blob[:-1])
    with pytest.raises(MalformedHeader):
        bl.deserialize_channel_int(blob)
    c = bl.ChannelIntPacket(shape=(2, 3), bits=4, scales=np.ones(3, np.float16),
                            code_stream=bytes(3))
    with pytest.raises(MalformedHeader):
        bl.deserialize_topk(bl.serialize_channel_int(c))
    with pytest.raises(TruncatedStream):
        bl.deserialize_channel_int(bl.serialize_channel_int(c)[:-1])
