"""GPU parity of the comparison codecs (TopK, channel-wise INT) against the
reference's own outputs (tests/golden/baselines.json) and the pinned
oracle (oracle/baselines_oracle.py)."""

import hashlib
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import baselines_oracle as BO  # noqa: E402
from tests.golden import inputs  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DT = {"bf16": torch.bfloat16, "f16": torch.float16, "f32": torch.float32}


def sha(b):
    if isinstance(b, np.ndarray):
        b = np.ascontiguousarray(b).tobytes()
    return hashlib.sha256(b).hexdigest()


@pytest.fixture(scope="module")
def bl():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2411_09510_b200 import baselines

    return baselines


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(ROOT, "tests", "golden", "baselines.json")) as f:
        return json.load(f)


def as_dtype(case):
    x = inputs.baseline_case(case)
    return x, torch.from_numpy(x).to(DT[inputs.BASELINE_CASES[case][1]])


CASES = list(inputs.BASELINE_CASES)


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("bits", [2, 3, 4, 5, 8])
def test_chanint_streams_bit_exact(bl, gold, case, bits):
    g = gold["chanint"][f"{case}|{bits}"]
    x64, xt = as_dtype(case)
    for inp in (xt.cuda(), x64):  # the kernel dtype and the reference's float64 input
        p = bl.channelwise_int_compress(inp, bits)
        sb = p.scales.astype("<f2").tobytes()
        assert g["scales"] in (sb.hex(), sha(sb)), case
        assert sha(p.code_stream) == g["codes"], case
        assert sha(bl.serialize_channel_int(p)) == g["container"]
        assert p.nbytes == g["nbytes"]
        dec = bl.channelwise_int_decompress(p)
        assert sha(dec.astype("<f8")) == g["dec64"], case
        q = bl.deserialize_channel_int(bl.serialize_channel_int(p))
        assert q.code_stream == p.code_stream and np.array_equal(q.scales, p.scales)


@pytest.mark.parametrize("case", CASES)
def test_topk_bit_exact(bl, gold, case):
    x64, xt = as_dtype(case)
    for key, g in gold["topk"].items():
        name, arg = key.split("|")
        if name != case:
            continue
        for inp in (xt.cuda(), x64):
            if "error" in g:
                with pytest.raises(Exception):
                    bl.topk_compress(inp, float(arg[1:]))
                continue
            p = (bl.topk_compress(inp, float(arg[1:])) if arg.startswith("f")
                 else bl.topk_compress(inp, k=int(arg[1:])))
            assert p.k_per_tensor == g["k"], key
            assert sha(p.indices.astype("<u4")) == g["indices"], key
            assert sha(p.values.astype("<f2")) == g["values"], key
            assert sha(bl.serialize_topk(p)) == g["container"], key
            if "dec64" in g:
                assert sha(bl.topk_decompress(p).astype("<f8")) == g["dec64"], key


def test_topk_random_vs_oracle(bl):
    """Many ties and every dtype: GPU == oracle (lexicographic (-|x|, index))."""
    rng = np.random.default_rng(5)
    for n, k in [(1, 1), (100, 100), (5000, 1), (5000, 2500), (70001, 777), (1 << 20, 99999)]:
        x = rng.choice(np.array([0.0, -0.0, 0.5, -0.5, 1.0, 2.0, -2.0, 3.0]), size=n)
        m = rng.random(n) < 0.3
        x[m] = rng.standard_normal(int(m.sum()))
        for dt in (torch.bfloat16, torch.float16, torch.float32):
            xt = torch.from_numpy(x).to(dt)
            ref_idx, ref_val = BO.topk_compress(xt.double().numpy(), k=k)
            p = bl.topk_compress(xt.cuda(), k=k)
            assert np.array_equal(p.indices, ref_idx), (n, k, dt)
            assert np.array_equal(p.values.view(np.uint16), ref_val.view(np.uint16)), (n, k, dt)


def test_chanint_random_vs_oracle(bl):
    rng = np.random.default_rng(6)
    for shape in [(1, 9), (7, 3), (300, 129), (64, 4096)]:
        x = (rng.standard_normal(shape) * 10.0 ** rng.uniform(-3, 3, size=shape[-1]))
        for dt in (torch.bfloat16, torch.float16, torch.float32):
            xt = torch.from_numpy(x).to(dt)
            x64 = xt.double().numpy()
            for bits in (2, 4, 7):
                s16, _, stream = BO.chanint_compress(x64, bits)
                p = bl.channelwise_int_compress(xt.cuda(), bits)
                assert np.array_equal(p.scales.view(np.uint16), s16.view(np.uint16))
                assert p.code_stream == stream, (shape, dt, bits)


def test_errors(bl):
    from paper_2411_09510_b200.errors import CompressionFactorTooHigh, NonFiniteInput

    with pytest.raises(CompressionFactorTooHigh):
        bl.topk_compress(np.ones(10), 1.0)
    with pytest.raises(CompressionFactorTooHigh):
        bl.topk_compress(np.ones(10), 3.0)  # budget < 1 value
    with pytest.raises(ValueError):
        bl.channelwise_int_compress(np.ones(4), 9)
    x = np.ones((4, 8))
    x[2, 3] = np.nan
    with pytest.raises(NonFiniteInput):
        bl.channelwise_int_compress(x, 4)
    with pytest.raises(NonFiniteInput):
        bl.topk_compress(x.ravel(), k=3)


def test_tpsim_baseline_codecs(gold):
    """simulate_reduction through topk / chanint / fp16 / passthrough ==
    the reference's report (mx/tpsim.py:234-302)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2411_09510_b200 import tp

    for g in gold["tpsim"]:
        cfg = tp.TPConfig(g["degree"], g["scheme"], g["seed"], tuple(g["input_shape"]),
                          tuple(g["weight_shape"]), g["quantize_own"])
        parts = [np.frombuffer(bytes.fromhex(h), dtype=np.float32).reshape(g["partial_shape"])
                 for h in g["partials_f32_hex"]]
        rep = tp.simulate_reduction(cfg, partials=parts)
        assert rep.scheme == g["name"]
        assert rep.rel_frob_err.hex() == g["rel_frob_err"], g["scheme"]
        assert rep.max_abs_err.hex() == g["max_abs_err"], g["scheme"]
        assert float(rep.sqnr_db).hex() == g["sqnr_db"], g["scheme"]
        assert (rep.bytes_compressed, rep.bytes_uncompressed, rep.padding) == (
            g["bytes_compressed"], g["bytes_uncompressed"], g["padding"])


@pytest.mark.parametrize("bits", [2, 3, 4, 5, 8])
def test_chanint_decompress_f32_bf16_vector_path(bl, bits):
    """f32 / bf16 outputs (vectorised decoder) equal the float64 decode
    rounded once (level * scale is exact in f32)."""
    rng = np.random.default_rng(40 + bits)
    x = rng.standard_normal((96, 256)) * 10.0 ** rng.uniform(-2, 2, size=256)
    x[:, 7] = 0.0
    s, c, shape = bl.channelwise_int_compress_device(torch.from_numpy(x).to("cuda", torch.float32),
                                                     bits)
    d64 = bl.channelwise_int_decompress_device(s, c, shape, bits, torch.float64).cpu().numpy()
    for dt in (torch.float32, torch.bfloat16):
        got = bl.channelwise_int_decompress_device(s, c, shape, bits, dt).cpu()
        want = torch.from_numpy(d64).to(dt)
        assert torch.equal(got.view(torch.int16 if dt == torch.bfloat16 else torch.int32),
                           want.view(torch.int16 if dt == torch.bfloat16 else torch.int32)), (bits, dt)
