"""GPU: the row-parallel GEMM with the MX quantiser fused into its epilogue
(k_gemm.cu: TMA -> tcgen05.mma into TMEM -> tcgen05.ld -> quantise).

Two properties, checked separately because the GEMM's fp32 accumulation
order is its own:
  * the GEMM: partial = x . w^T against a float64 reference of the same bf16
    operands, within a stated tolerance (fp32 accumulation over K terms, one
    bf16 rounding);
  * the quantiser: the shard bytes the epilogue writes are byte-identical to
    the oracle's compress() of the SAME kernel call's bf16 partial
    (mx/codec.py:238-263) -- the exactness bar of K1.
Then the collective wiring: CompressedAllReduce.linear at world 1 and at
N = 2 / 4 ranks (LocalThreadGroup, one device) equals quantising that
partial through the unfused path (mx/tpsim.py:263-265 hook order).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import mx_oracle as O  # noqa: E402


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2411_09510_b200 import _native

    return _native.load()


def operands(M, N, K, seed, std=1.0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    x = (torch.randn(M, K, generator=g) * std).to(torch.bfloat16)
    w = (torch.randn(N, K, generator=g) / K ** 0.5).to(torch.bfloat16)
    # a few large outliers (activation-like), so blocks use several exponents
    x.view(-1)[:: 997] *= 64
    return x.cuda(), w.cuda()


def gemm(lib, x, w, spec=None, partial=True):
    import ctypes

    from paper_2411_09510_b200 import _native
    from paper_2411_09510_b200.formats import parse_scheme

    M, K = x.shape
    N = w.shape[0]
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    part = torch.empty(M, N, dtype=torch.bfloat16, device="cuda") if partial else None
    if spec is None:
        _native.check(lib.mx_gemm_quantize(
            ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(w.data_ptr()), M, N, K, None, None,
            None, ctypes.c_void_p(part.data_ptr()), None, st), "mx_gemm_quantize")
        return part, None, None, None
    cs = parse_scheme(spec, extensions=True).to_c()
    sb, eb = _native.stream_nbytes(M * N, cs)
    sc = torch.empty(sb, dtype=torch.uint8, device="cuda")
    el = torch.empty(eb, dtype=torch.uint8, device="cuda")
    flag = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    _native.check(lib.mx_gemm_quantize(
        ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(w.data_ptr()), M, N, K, ctypes.byref(cs),
        ctypes.c_void_p(sc.data_ptr()), ctypes.c_void_p(el.data_ptr()),
        ctypes.c_void_p(part.data_ptr()) if part is not None else None,
        ctypes.c_void_p(flag.data_ptr()), st), "mx_gemm_quantize")
    return part, sc, el, flag


def check_gemm(x, w, part):
    """|ours - ref| <= 2^-8 |ref| + 2^-20 K max|x||w| : one bf16 rounding of
    the result plus fp32 accumulation error over K terms."""
    ref = x.double() @ w.double().T
    got = part.double()
    bound = ref.abs() * 2.0 ** -8 + 2.0 ** -20 * x.shape[1] * x.double().abs().max() * \
        w.double().abs().max()
    bad = (got - ref).abs() > bound
    assert not bool(bad.any()), f"{int(bad.sum())} values outside the GEMM tolerance"


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 512, 512), (200, 384, 192),
                                   (1024, 4096, 1024), (333, 128, 2048)])
def test_plain_gemm_matches_float64(lib, M, N, K):
    x, w = operands(M, N, K, seed=M + N + K)
    part, _, _, _ = gemm(lib, x, w)
    torch.cuda.synchronize()
    check_gemm(x, w, part)
    # cuBLAS agrees to the same tolerance (sanity on the reference itself)
    check_gemm(x, w, torch.nn.functional.linear(x, w))


@pytest.mark.parametrize("spec", ["fp4_e2m1:32:e8m0", "fp4_e2m1:16:e8m0", "fp6_e2m3:32:e8m0",
                                  "fp6_e3m2:32:e8m0", "fp5_e2m2:32:e8m0", "int8:32:e8m0",
                                  "int8:16:e8m0", "fp4_e2m1:8:e8m0",
                                  # E5M0: the paper's selected schemes (N % 256 == 0)
                                  "fp4_e2m1:8:e5m0", "fp4_e2m1:16:e5m0", "fp4_e2m1:32:e5m0",
                                  "fp5_e2m2:32:e5m0"])
@pytest.mark.parametrize("M,N,K", [(256, 512, 256), (200, 384, 128), (1152, 2048, 512)])
def test_fused_quantiser_bytes_equal_oracle(lib, spec, M, N, K):
    if spec.endswith("e5m0") and N % 256:
        pytest.skip("E5M0 GEMM epilogue needs N % 256 == 0 (falls back to F.linear + K1)")
    x, w = operands(M, N, K, seed=7 * M + K)
    part, sc, el, flag = gemm(lib, x, w, spec)
    torch.cuda.synchronize()
    check_gemm(x, w, part)
    flat = part.float().cpu().numpy().ravel().astype(np.float64)
    ss, es = O.compress(flat, O.scheme(spec))
    assert bytes(sc.cpu().numpy()) == ss, spec
    assert bytes(el.cpu().numpy()) == es, spec
    assert int(flag.item()) == -1
    # without the partial output the shard is the same
    _, sc2, el2, _ = gemm(lib, x, w, spec, partial=False)
    assert torch.equal(sc, sc2) and torch.equal(el, el2)


def test_fused_quantiser_8b_oproj_shape(lib):
    """Llama-3.1-8B o_proj at TP=2: [2048 x 2048] . [4096 x 2048]^T (more
    tiles than SMs: the persistent loop and both TMEM accumulators)."""
    spec = "fp4_e2m1:32:e8m0"
    x, w = operands(2048, 4096, 2048, seed=11)
    part, sc, el, _ = gemm(lib, x, w, spec)
    torch.cuda.synchronize()
    check_gemm(x, w, part)
    ss, es = O.compress(part.float().cpu().numpy().ravel().astype(np.float64), O.scheme(spec))
    assert bytes(sc.cpu().numpy()) == ss and bytes(el.cpu().numpy()) == es


def test_nonfinite_flag(lib):
    spec = "fp4_e2m1:32:e8m0"
    M, N, K = 256, 256, 128
    x, w = operands(M, N, K, seed=3)
    x[37, 5] = float("nan")
    _, _, _, flag = gemm(lib, x, w, spec)
    torch.cuda.synchronize()
    assert int(flag.item()) == 37 * N  # first non-finite flat index (row 37, column 0)


def test_unsupported_shapes_raise(lib):
    x, w = operands(128, 200, 64, seed=1)  # N % 128 != 0
    with pytest.raises(Exception, match="fused GEMM"):
        gemm(lib, x, w, "fp4_e2m1:32:e8m0")
    x, w = operands(128, 256, 96, seed=1)  # K % 64 != 0
    with pytest.raises(Exception, match="fused GEMM"):
        gemm(lib, x, w)


@pytest.mark.parametrize("algo", ["oneshot", "twoshot"])
def test_collective_linear_world1(lib, algo):
    from paper_2411_09510_b200.collective import CompressedAllReduce

    spec = "fp4_e2m1:32:e8m0"
    M, N, K = 512, 1024, 256
    x, w = operands(M, N, K, seed=5)
    part, _, _, _ = gemm(lib, x, w)  # the same GEMM's bf16 partial
    car = CompressedAllReduce(spec, M * N, algo=algo, out_dtype=torch.bfloat16)
    got = car.linear(x, w).clone()
    want = car(part).clone()
    torch.cuda.synchronize()
    assert got.shape == (M, N)
    assert torch.equal(got.view(torch.int16), want.view(torch.int16))


@pytest.mark.parametrize("spec", ["fp4_e2m1:32:e8m0", "fp4_e2m1:8:e5m0", "fp5_e2m2:32:e5m0"])
@pytest.mark.parametrize("N", [2, 4])
@pytest.mark.parametrize("algo", ["oneshot", "twoshot"])
def test_collective_linear_multirank(lib, N, algo, spec):
    """N ranks (threads, LocalThreadGroup): each rank's fused GEMM shard goes
    through the real exchange; every rank equals the oracle's all-reduce of
    the ranks' bf16 partials (the same kernels' plain-mode output)."""
    from paper_2411_09510_b200.collective import CompressedAllReduce, LocalThreadGroup

    M, Nout, K = 256, 1024, 256
    ops = [operands(M, Nout, K, seed=40 + r) for r in range(N)]
    parts = [gemm(lib, x, w)[0] for x, w in ops]
    torch.cuda.synchronize()
    host = [p.float().cpu().numpy().ravel().astype(np.float64) for p in parts]
    osch = O.scheme(spec)
    ref = (O.allreduce_oneshot if algo == "oneshot" else O.allreduce_twoshot)(host, osch)
    want = torch.from_numpy(np.asarray(ref, np.float32)).to(torch.bfloat16).view(torch.int16)
    grp = LocalThreadGroup(N)

    def rank_fn(r):
        car = CompressedAllReduce(spec, M * Nout, algo=algo, out_dtype=torch.bfloat16, comm=grp)
        x, w = ops[r]
        return car.linear(x, w).reshape(-1).view(torch.int16).cpu()

    for r, o in enumerate(grp.run(rank_fn)):
        assert torch.equal(o, want), (N, algo, r)


def test_row_parallel_linear_uses_fused_gemm(lib, monkeypatch):
    """RowParallelLinear (the TP model hook) routes through the fused GEMM
    by default and through F.linear + K1 with MXB200_GEMM_FUSED=0; both
    reduce the same partial up to the GEMM's own accumulation order, so
    compare each against its own partial."""
    from paper_2411_09510_b200 import tp

    RPL = tp.make_module_classes()[0]
    lin = RPL(256, 512, scheme="fp4_e2m1:32:e8m0", algo="oneshot", device="cuda")
    assert lin.fused_gemm
    x = torch.randn(2, 64, 256, device="cuda").to(torch.bfloat16)
    y = lin(x)
    part, _, _, _ = gemm(lib, x.reshape(128, 256), lin.weight.data)
    car = lin._collective(128 * 512, torch.bfloat16, x.device)
    want = car(part.clone()).clone()
    assert y.shape == (2, 64, 512)
    assert torch.equal(y.reshape(-1).view(torch.int16), want.reshape(-1).view(torch.int16))
    lin.fused_gemm = False
    y2 = lin(x)
    ref = torch.nn.functional.linear(x, lin.weight)
    want2 = car(ref.reshape(-1).contiguous()).clone()
    assert torch.equal(y2.reshape(-1).view(torch.int16), want2.reshape(-1).view(torch.int16))
