"""GPU parity: the sm_100a kernels (through the C ABI) vs the pinned oracle.

Bit-exact everywhere: scale streams, element streams, fp32 / fp64
decompression, fp32 rank-order sums and their bf16 cast.  The golden
digests were produced by the real reference (tests/golden/make_golden.py)
and the oracle is pinned to the same digests (tests/test_oracle_golden.py),
so a match here is a match with mxcomm itself.
"""

import hashlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import mx_oracle as O  # noqa: E402
from tests.golden import inputs  # noqa: E402


def sha(b):
    if isinstance(b, np.ndarray):
        b = np.ascontiguousarray(b).tobytes()
    return hashlib.sha256(b).hexdigest()


@pytest.fixture(scope="module")
def mx():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2411_09510_b200 as m
    from paper_2411_09510_b200 import _native

    _native.load()
    return m


TORCH_DT = {"bf16": torch.bfloat16, "f16": torch.float16, "f32": torch.float32,
            "f64": torch.float64}


def dev(x64, dtype):
    t = torch.from_numpy(np.asarray(x64, dtype=np.float64))
    return t.to(TORCH_DT[dtype]).cuda()


def scheme_of(mx, spec):
    return mx.parse_scheme(spec, extensions=True)


def gpu_streams(mx, x, sch):
    dct = mx.compress_tensor_device(x, sch)
    return dct.scale.cpu().numpy().tobytes(), dct.elements.cpu().numpy().tobytes(), dct


# ---------------------------------------------------------------------------


def test_explicit_vectors(mx, golden):
    for v in golden["vectors"]:
        sch = scheme_of(mx, v["scheme"])
        x = np.array([float.fromhex(h) for h in v["values_hex"]])
        ct = mx.compress_tensor(x, sch)  # float64 numpy input: generic kernels
        assert ct.scale_stream.hex() == v["scale_stream"], v["name"]
        assert ct.element_stream.hex() == v["element_stream"], v["name"]
        dec = mx.decompress_tensor(ct)
        assert [float(d).hex() for d in dec] == v["decoded_hex"], v["name"]
        if np.array_equal(x.astype(np.float32).astype(np.float64), x):  # f32 fast path too
            ss, es, _ = gpu_streams(mx, dev(x, "f32"), sch)
            assert ss.hex() == v["scale_stream"] and es.hex() == v["element_stream"], v["name"]


@pytest.mark.parametrize("case", list(inputs.CASES))
def test_digest_sweep(mx, golden, case):
    gen, dtype = inputs.CASES[case]
    x64 = gen()
    x = dev(x64, dtype)
    g = golden["digests"][case]
    bad = []
    for spec, d in g["schemes"].items():
        sch = scheme_of(mx, spec)
        ss, es, dct = gpu_streams(mx, x, sch)
        if sha(ss) != d["scale"] or sha(es) != d["elem"]:
            oss, oes = O.compress(x64, O.scheme(spec))
            first = next((i for i, (a, b) in enumerate(zip(es, oes)) if a != b), None)
            bad.append(f"{spec}: scale_ok={sha(ss) == d['scale']} elem_ok={sha(es) == d['elem']}"
                       f" first_elem_byte_diff={first}")
            continue
        d32 = mx.decompress_tensor_device(dct, torch.float32).cpu().numpy()
        if sha(d32) != d["dec32"]:
            bad.append(spec + "/dec32")
        d64 = mx.decompress_tensor_device(dct, torch.float64).cpu().numpy()
        if sha(d64) != d["dec64"]:
            bad.append(spec + "/dec64")
    assert not bad, bad


def test_float64_and_unaligned_inputs_take_generic_path(mx, golden):
    x64 = inputs.gauss_f32(5003, 4)
    d = golden["digests"]["gauss_f32_5003"]["schemes"]
    for spec in ["fp4_e2m1:32:e8m0", "fp5_e3m1:32:e5m0", "int8:64:e8m0", "fp4_e2m1:7:e8m0"]:
        sch = scheme_of(mx, spec)
        ss, es, _ = gpu_streams(mx, dev(x64, "f64"), sch)
        assert sha(ss) == d[spec]["scale"] and sha(es) == d[spec]["elem"], spec
        # misaligned (offset by one element) bf16/f32 views
        buf = torch.zeros(x64.size + 1, dtype=torch.float32, device="cuda")
        buf[1:] = dev(x64, "f32")
        ss, es, _ = gpu_streams(mx, buf[1:], sch)
        assert sha(ss) == d[spec]["scale"] and sha(es) == d[spec]["elem"], spec + " unaligned"


def test_decode_random_streams(mx, golden):
    bad = []
    for spec, d in golden["decode"].items():
        sch = scheme_of(mx, spec)
        n = d["n"]
        nb = -(-n // sch.block_size)
        ss, es = inputs.random_streams((nb * sch.scale.exponent_bits + 7) // 8,
                                       (n * sch.element.total_bits + 7) // 8, d["seed"])
        ct = mx.CompressedTensor(sch, (n,), ss, es)
        if sha(mx.decompress_tensor(ct, np.float32)) != d["dec32"]:
            bad.append(spec)
        if sha(mx.decompress_tensor(ct, np.float64)) != d["dec64"]:
            bad.append(spec + "/64")
    assert not bad, bad


def test_rank_order_reduction_oneshot(mx, golden):
    from paper_2411_09510_b200.collective import simulate_allreduce

    for spec, d in golden["reduce"].items():
        parts = [dev(inputs.gauss_bf16(d["n"], s), "bf16") for s in d["seeds"]]
        out32, _ = simulate_allreduce(parts, spec, "oneshot", torch.float32)
        assert sha(out32.cpu().numpy()) == d["sum32"], spec
        out16, _ = simulate_allreduce(parts, spec, "oneshot", torch.bfloat16)
        ref16 = O.to_bf16_bits(out32.cpu().numpy())
        assert np.array_equal(out16.cpu().view(torch.int16).numpy().view(np.uint16), ref16), spec


@pytest.mark.parametrize("N", [2, 3, 4, 8])
@pytest.mark.parametrize("spec", ["fp4_e2m1:32:e8m0", "fp5_e2m2:16:e8m0", "fp6_e2m3:64:e8m0",
                                  "int8:32:e8m0", "fp4_e2m1:8:e5m0", "fp4_e2m1:24:e8m0"])
def test_oneshot_and_twoshot_vs_oracle(mx, N, spec):
    from paper_2411_09510_b200.collective import simulate_allreduce

    n = 70001
    x64 = [inputs.gauss_bf16(n, 1000 + r) for r in range(N)]
    parts = [dev(x, "bf16") for x in x64]
    osch = O.scheme(spec)
    one, _ = simulate_allreduce(parts, spec, "oneshot", torch.float32)
    assert np.array_equal(one.cpu().numpy(), O.allreduce_oneshot(x64, osch)), "oneshot"
    two, _ = simulate_allreduce(parts, spec, "twoshot", torch.float32)
    ref2 = O.allreduce_twoshot(x64, osch)
    assert np.array_equal(two.cpu().numpy(), ref2), "twoshot"
    # two-shot error vs one-shot is bounded by one requantisation step
    st, _ = O.quantize(ref2.astype(np.float64), osch)
    bound = np.array([mx.block_error_bound(int(s), scheme_of(mx, spec)) for s in st])
    per = np.repeat(bound, osch.block)[:n]
    assert np.all(np.abs(ref2.astype(np.float64) - one.cpu().numpy()) <= per * 1.0000001 + 1e-30)


@pytest.mark.parametrize("N", [2, 4, 8])
@pytest.mark.parametrize("spec", ["fp4_e2m1:32:e8m0", "fp6_e2m3:64:e8m0", "int8:16:e8m0",
                                  "fp4_e2m1:8:e5m0", "fp5_e2m2:32:e5m0"])
def test_twoshot_whole_unit_chunks_vs_oracle(mx, N, spec):
    """Chunk sizes that are multiples of 1024 take the chunked full-unit K1
    path and the multi-chunk lean K2; both must stay bit-exact."""
    from paper_2411_09510_b200.collective import simulate_allreduce

    n = 1 << 18
    x64 = [inputs.gauss_bf16(n, 3100 + r) for r in range(N)]
    parts = [dev(x, "bf16") for x in x64]
    osch = O.scheme(spec)
    for out_dt in (torch.float32, torch.bfloat16):
        two, _ = simulate_allreduce(parts, spec, "twoshot", out_dt)
        ref = O.allreduce_twoshot(x64, osch)
        got = two.float().cpu().numpy()
        want = torch.from_numpy(ref).to(out_dt).float().numpy()
        assert np.array_equal(got, want), (spec, N, out_dt)


def test_large_prefill_shape_tp2(mx, golden):
    from paper_2411_09510_b200.collective import simulate_allreduce
    from paper_2411_09510_b200.synth import rank_partials

    g = golden["large"]
    p0, p1 = rank_partials(tuple(g["shape"]), 2, seed=0)
    assert [sha(p0), sha(p1)] == g["input_sha"]
    t0, t1 = dev(p0, "bf16"), dev(p1, "bf16")
    for spec in inputs.LARGE_SCHEMES:
        sch = scheme_of(mx, spec)
        ss, es, _ = gpu_streams(mx, t0, sch)
        assert sha(ss) == g[spec]["scale"] and sha(es) == g[spec]["elem"], spec
        out, _ = simulate_allreduce([t0, t1], spec, "oneshot", torch.float32)
        assert sha(out.cpu().numpy()) == g[spec]["tp2_sum32"], spec


def test_nonfinite_block_index(mx, golden):
    for d in golden["nonfinite"]:
        x = np.ones(4099)
        x[d["index"]] = float(d["value"])
        x[4098] = np.nan
        for dtype in ["f32", "bf16", "f64"]:
            with pytest.raises(mx.NonFiniteInput) as ei:
                mx.compress_tensor(dev(x, dtype), scheme_of(mx, f"fp4_e2m1:{d['block']}:e8m0"))
            assert ei.value.block_index == d["block_index"], (d, dtype)


def test_chunked_quantize_equals_whole_tensor(mx):
    from paper_2411_09510_b200 import _native
    import ctypes

    x64 = inputs.gauss_bf16(100000, 21)
    x = dev(x64, "bf16")
    for spec in ["fp4_e2m1:32:e8m0", "fp5_e3m1:16:e6m0", "int8:64:e8m0"]:
        sch = scheme_of(mx, spec)
        cs = sch.to_c()
        c = 8 * sch.block_size * 37
        so, eo, S = _native.shard_layout(c, cs)
        nch = -(-x.numel() // c)
        shards = torch.zeros(nch * S, dtype=torch.uint8, device="cuda")
        ws = torch.empty(_native.workspace_bytes(nch * c, cs), dtype=torch.uint8, device="cuda")
        lib = _native.load()
        _native.check(lib.mx_quantize_chunks(
            ctypes.c_void_p(x.data_ptr()), _native.MX_BF16, x.numel(), c, ctypes.byref(cs),
            ctypes.c_void_p(shards.data_ptr()), S, None, ctypes.c_void_p(ws.data_ptr()),
            ws.numel(), None), "chunks")
        host = shards.cpu().numpy()
        ss, es = O.compress(x64, O.scheme(spec))
        sb_c = c // sch.block_size * sch.scale.exponent_bits // 8
        eb_c = c * sch.element.total_bits // 8
        got_s = b"".join(host[j * S + so: j * S + so + sb_c].tobytes() for j in range(nch))
        got_e = b"".join(host[j * S + eo: j * S + eo + eb_c].tobytes() for j in range(nch))
        assert got_s[:len(ss)] == ss and got_e[:len(es)] == es, spec


def test_block_api(mx):
    sch = scheme_of(mx, "fp4_e2m1:32:e8m0")
    stored, codes = mx.quantize_block([1.0, -6.0, 0.25, 3.0], sch)
    assert stored == 127 and codes.tolist() == [2, 15, 0, 5]
    assert mx.dequantize_block(stored, codes, sch).tolist() == [1.0, -6.0, 0.0, 3.0]
    stored, codes = mx.quantize_block([2.0 ** 130, 1.0], scheme_of(mx, "fp4_e2m1:32:e5m0"))
    assert stored == 31 and codes.tolist() == [7, 0]
    with pytest.raises(mx.MalformedCode):
        mx.dequantize_block(127, [16], sch)
    with pytest.raises(ValueError):
        mx.quantize_block(np.zeros(33), sch)


def test_serialize_roundtrip_on_gpu_streams(mx):
    sch = scheme_of(mx, "fp4_e2m1:32:e8m0")
    x = inputs.gauss_bf16(2 * 128 * 64, 7).reshape(2, 128, 64)
    ct = mx.compress_tensor(x, sch)
    blob = mx.serialize(ct)
    assert len(blob) == mx.serialized_nbytes(sch, x.shape) == 44 + 512 + 8192
    back = mx.deserialize(blob)
    assert back == ct
    assert np.array_equal(mx.decompress_tensor(back), O.decompress(
        ct.scale_stream, ct.element_stream, x.size, O.scheme(sch.name)).reshape(x.shape))


def test_empty_and_tiny(mx):
    sch = scheme_of(mx, "fp4_e2m1:32:e8m0")
    ct = mx.compress_tensor(np.zeros((0,)), sch)
    assert ct.scale_stream == b"" and ct.element_stream == b""
    assert mx.decompress_tensor(ct).shape == (0,)
    ct = mx.compress_tensor(np.float64(3.0), sch)  # 0-d tensor: one value
    assert mx.decompress_tensor(ct).shape == () and float(mx.decompress_tensor(ct)) == 3.0


@pytest.mark.parametrize("spec", ["fp4_e2m1:32:e8m0", "fp4_e2m1:8:e8m0", "fp6_e2m3:64:e8m0",
                                  "int8:16:e8m0", "fp5_e2m2:32:e8m0",
                                  # packed k-bit scales: the paper's selected schemes (lean
                                  # K1/K2/K4 with S8 = false) and a format without a lean
                                  # k-bit instantiation (general kernels)
                                  "fp4_e2m1:8:e5m0", "fp5_e2m2:32:e5m0", "fp4_e2m1:64:e5m0",
                                  "fp4_e2m1:16:e4m0", "fp6_e2m3:32:e5m0"])
@pytest.mark.parametrize("N", [1, 2, 3, 8])
def test_fused_oneshot_bit_identical(mx, spec, N):
    """One persistent kernel (quantise, grid barrier, dequant-sum) == the
    separate K1 x N + K2 launches == the oracle."""
    from paper_2411_09510_b200.collective import SimulatedAllReduce

    for n in (1 << 20, 70001):
        x64 = [inputs.gauss_bf16(n, 2000 + r) for r in range(N)]
        parts = [dev(x, "bf16") for x in x64]
        fused = SimulatedAllReduce(spec, n, N, "oneshot", torch.float32, fused=True)
        split = SimulatedAllReduce(spec, n, N, "oneshot", torch.float32, fused=False)
        a = fused(parts).cpu().numpy().copy()
        a2 = fused(parts).cpu().numpy().copy()  # barrier reuse across calls
        b = split(parts).cpu().numpy()
        assert fused.fused, "fused kernel not taken"
        assert np.array_equal(a, b) and np.array_equal(a, a2)
        assert np.array_equal(a, O.allreduce_oneshot(x64, O.scheme(spec)))


def test_tma_quantiser_opt_in_bit_exact(mx):
    """K1's opt-in TMA pipeline (MXB200_TMA=1; read once per process, so a
    subprocess) writes the same streams as the oracle, whole tiles plus a
    register-path remainder."""
    import os
    import subprocess
    import sys

    code = r"""
import numpy as np, torch
from oracle import mx_oracle as O
from tests.golden import inputs
import paper_2411_09510_b200 as mx
for n, spec in [(8192 * 3 + 1000, "fp4_e2m1:32:e8m0"), (8192 * 5, "fp6_e2m3:16:e8m0"),
                (8192 * 2 + 64, "int8:64:e8m0")]:
    x64 = inputs.gauss_bf16(n, 77)
    d = mx.compress_tensor_device(torch.from_numpy(x64).to("cuda", torch.bfloat16),
                                  mx.parse_scheme(spec, extensions=True))
    ss, es = O.compress(x64, O.scheme(spec))
    assert d.scale.cpu().numpy().tobytes() == ss, spec
    assert d.elements.cpu().numpy().tobytes() == es, spec
print("tma ok")
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MXB200_TMA="1", PYTHONPATH=root)
    p = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                       text=True, timeout=300)
    assert p.returncode == 0 and "tma ok" in p.stdout, p.stderr[-2000:]


@pytest.mark.parametrize("spec", ["fp4_e2m1:32:e8m0", "fp3_e1m1:32:e8m0", "int5:16:e8m0",
                                  "fp6_e3m2:64:e8m0"])
@pytest.mark.parametrize("n", [1024, 4096, 5 * 1024, 12288])
@pytest.mark.parametrize("fused", [True, False])
def test_unit_counts_not_multiple_of_cta(mx, spec, n, fused):
    """Sizes whose 1024-value unit count is not a multiple of the 8 warps of
    a CTA (the lean kernels' grid must round up); bit-level comparison,
    including the sign of zero, one-shot and two-shot."""
    from paper_2411_09510_b200.collective import SimulatedAllReduce

    for N, algo in ((2, "oneshot"), (3, "oneshot"), (2, "twoshot"), (4, "twoshot")):
        x64 = [inputs.gauss_bf16(n, 7100 + N + r) for r in range(N)]
        for x in x64:
            x[::97] = 0.0
        parts = [dev(x, "bf16") for x in x64]
        op = SimulatedAllReduce(spec, n, N, algo, torch.float32,
                                fused=fused and algo == "oneshot")
        got = op(parts).cpu().numpy()
        ref = (O.allreduce_oneshot if algo == "oneshot" else O.allreduce_twoshot)(
            x64, O.scheme(spec))
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), (spec, n, N, algo)
