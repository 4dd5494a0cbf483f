"""GPU: the Llama residual update fused into the compressed all-reduce's
dequant-sum store (``mx_dequant_sum_residual`` / the ``residual`` argument
of ``CompressedAllReduce`` and ``RowParallelLinear``).

The bar is bit-identity with the unfused sequence the reference hook
implies -- the all-reduced tensor in out_dtype (mx/tpsim.py:263-281,
mx/netbench.py:332-334), then ``h + y`` as an elementwise add in out_dtype
-- for every kernel path (lean K2, general K2 on ragged sizes, generic
K2 for odd block sizes), both algorithms, N = 1..4 ranks, in-place
(``out`` is the residual) and out of place."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import mx_oracle as O  # noqa: E402
from tests.golden import inputs  # noqa: E402


@pytest.fixture(scope="module")
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2411_09510_b200 import _native

    _native.load()
    return torch.device("cuda", 0)


CASES = [("fp4_e2m1:32:e8m0", 8192), ("fp4_e2m1:32:e8m0", 5003), ("fp5_e2m2:16:e5m0", 3000),
         ("int8:64:e8m0", 4096 + 64), ("fp4_e2m1:24:e8m0", 2400)]


def _run(parts, spec, algo, out_dtype, resid, inplace):
    from paper_2411_09510_b200.collective import CompressedAllReduce, LocalThreadGroup

    N = len(parts)
    grp = LocalThreadGroup(N) if N > 1 else None

    def rank_fn(r):
        car = CompressedAllReduce(spec, parts[r].numel(), algo=algo, out_dtype=out_dtype,
                                  comm=grp)
        h = resid[r].clone()
        out = car(parts[r], out=h if inplace else None, residual=h)
        if inplace:
            assert out.data_ptr() == h.data_ptr()
        car.check_finite()
        return out.clone()

    return grp.run(rank_fn) if grp is not None else [rank_fn(0)]


@pytest.mark.parametrize("N", [1, 2, 4])
@pytest.mark.parametrize("algo", ["oneshot", "twoshot"])
@pytest.mark.parametrize("out_dtype", [torch.bfloat16, torch.float32])
def test_residual_fused_equals_add(cuda, N, algo, out_dtype):
    for spec, n in CASES:
        x64 = [inputs.gauss_bf16(n, 700 + r) for r in range(N)]
        parts = [torch.from_numpy(x).to(cuda, torch.bfloat16) for x in x64]
        resid = [torch.from_numpy(inputs.gauss_bf16(n, 800 + r)).to(cuda, out_dtype)
                 for r in range(N)]
        f = O.allreduce_oneshot if algo == "oneshot" else O.allreduce_twoshot
        s = torch.from_numpy(np.asarray(f(x64, O.scheme(spec)), np.float32)).to(cuda, out_dtype)
        for inplace in (False, True):
            got = _run(parts, spec, algo, out_dtype, resid, inplace)
            for r in range(N):
                want = resid[r] + s
                assert torch.equal(got[r], want), (spec, n, algo, N, r, inplace)


def test_residual_rejects_mismatch(cuda):
    from paper_2411_09510_b200.collective import CompressedAllReduce
    from paper_2411_09510_b200.errors import ShapeMismatch

    car = CompressedAllReduce("fp4_e2m1:32:e8m0", 4096, out_dtype=torch.bfloat16)
    x = torch.randn(4096, device=cuda).to(torch.bfloat16)
    with pytest.raises(ShapeMismatch):
        car(x, residual=torch.zeros(4096, device=cuda, dtype=torch.float32))
    with pytest.raises(ShapeMismatch):
        car(x, residual=torch.zeros(4095, device=cuda, dtype=torch.bfloat16))


@pytest.mark.parametrize("fused_gemm", [False, True])
def test_row_parallel_linear_residual(cuda, fused_gemm, monkeypatch):
    """RowParallelLinear(x, residual=h) with the add fused into K2 == the
    same layer with the add after the collective (MXB200_FUSE_RESIDUAL=0)."""
    from paper_2411_09510_b200.tp import make_module_classes

    RowParallelLinear = make_module_classes()[0]
    torch.manual_seed(0)
    x = torch.randn(2, 128, 512, device=cuda).to(torch.bfloat16)
    h = torch.randn(2, 128, 1024, device=cuda).to(torch.bfloat16)
    lin = RowParallelLinear(512, 1024, scheme="fp4_e2m1:32:e8m0", device=cuda,
                            fused_gemm=fused_gemm)
    assert lin.fuse_residual
    fused = lin(x, residual=h).clone()
    lin.fuse_residual = False
    unfused = lin(x, residual=h).clone()
    plain = h + lin(x)
    assert torch.equal(fused, unfused)
    assert torch.equal(fused, plain)


@pytest.mark.parametrize("algo", ["oneshot", "twoshot"])
def test_llama_shared_collectives_equal_per_layer(cuda, algo):
    """LlamaTP shares one collective buffer set across its layers (the
    residual-fused reduce updates h in place); the forward must equal the
    same model with a private buffer set per layer, bit for bit."""
    from paper_2411_09510_b200 import tp

    LlamaTP = tp.make_module_classes()[3]
    cfg = tp.LlamaConfig(512, 1024, 2, 8, 4)
    torch.manual_seed(1)
    model = LlamaTP(cfg, 1, None, "fp4_e2m1:32:e8m0", algo, device=cuda)
    h = torch.randn(1, 256, cfg.hidden, device=cuda).to(torch.bfloat16)
    with torch.inference_mode():
        shared = model(h).clone()
        assert len({id(c) for c in model.collectives()}) == 1
        for blk in model.blocks:
            for m in (blk.o_proj, blk.down_proj):
                m._shared, m._car = None, {}
        private = model(h).clone()
        assert len({id(c) for c in model.collectives()}) == 2 * len(model.blocks)
    assert torch.equal(shared, private)
