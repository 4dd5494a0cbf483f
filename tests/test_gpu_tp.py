"""GPU tests of the row-parallel hook: the simulated reduction reproduces the
reference's reports exactly (mx/tpsim.py:234-302), and the TP Llama harness
runs with the compressed all-reduce in place of NCCL bf16."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tp():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2411_09510_b200 import tp as m

    return m


def test_simulate_reduction_matches_reference(tp, golden):
    for g in golden["tpsim"]:
        cfg = tp.TPConfig(g["degree"], g["scheme"], g["seed"], tuple(g["input_shape"]),
                          tuple(g["weight_shape"]), g["quantize_own"])
        parts = [np.frombuffer(bytes.fromhex(h), dtype=np.float32).reshape(g["partial_shape"])
                 for h in g["partials_f32_hex"]]
        rep = tp.simulate_reduction(cfg, partials=parts)
        assert rep.rel_frob_err.hex() == g["rel_frob_err"], g
        assert rep.max_abs_err.hex() == g["max_abs_err"], g
        assert float(rep.sqnr_db).hex() == g["sqnr_db"], g
        assert (rep.bytes_compressed, rep.bytes_uncompressed, rep.padding) == (
            g["bytes_compressed"], g["bytes_uncompressed"], g["padding"])


def test_parallelism_sweep_triangle_bound(tp):
    reps = tp.parallelism_sweep(tp.TPConfig(2, "fp4_e2m1:32:e8m0", 7, (1, 32, 512), (512, 256)),
                                [2, 4, 8, 16])
    assert [r.degree for r in reps] == [2, 4, 8, 16]
    assert all(0 < r.rel_frob_err < 0.5 for r in reps)


def test_row_parallel_linear_single_rank(tp):
    RowParallelLinear, _, _, _ = tp.make_module_classes()
    torch.manual_seed(0)
    lin = RowParallelLinear(512, 256, scheme="fp4_e2m1:32:e8m0")
    x = torch.randn(4, 64, 512, device="cuda", dtype=torch.bfloat16)
    y = lin(x)
    ref = torch.nn.functional.linear(x, lin.weight).float()
    # one rank: output = decode(quantise(partial)), error bounded per block
    err = (y.float() - ref).abs().max().item()
    assert err <= ref.abs().max().item() * 0.25 + 1e-3
    assert y.shape == (4, 64, 256) and y.dtype == torch.bfloat16


def test_llama_tp_prefill_smoke(tp):
    cfg = tp.LlamaConfig(hidden=512, ffn=1536, layers=2, heads=8, kv_heads=2)
    ms_bf16 = tp.measure_ttft(cfg, batch=1, seq=128, tp=1, scheme=None, reps=2, warmup=1)
    ms_mx = tp.measure_ttft(cfg, batch=1, seq=128, tp=1, scheme="fp4_e2m1:32:e8m0", reps=2,
                            warmup=1)
    assert ms_bf16 > 0 and ms_mx > 0
