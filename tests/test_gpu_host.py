"""Host-buffer path (HostPipeline) and the barrier-free fused kernel.

HostPipeline cuts the tensor into 1024-aligned pieces and overlaps their
H2D copies, compressed all-reduce and D2H copies on three streams; the host
result must equal the whole-tensor device call and the oracle bit for bit.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import mx_oracle as O  # noqa: E402
from tests.golden import inputs  # noqa: E402


@pytest.fixture(scope="module")
def coll():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2411_09510_b200 import collective

    return collective


def _bf16(x64):
    return torch.from_numpy(np.asarray(x64, dtype=np.float64)).to(torch.bfloat16)


@pytest.mark.parametrize("spec", ["fp4_e2m1:32:e8m0", "fp6_e2m3:16:e8m0"])
@pytest.mark.parametrize("N,n,chunks", [(2, 1 << 20, 8), (3, 8 * 4096, 4), (2, 5 * 1024, 8)])
def test_host_pipeline_bit_exact(coll, spec, N, n, chunks):
    x64 = [inputs.gauss_bf16(n, 500 + r) for r in range(N)]
    host = [_bf16(x).pin_memory() for x in x64]
    out = torch.empty(n, dtype=torch.float32).pin_memory()
    pipe = coll.HostPipeline.simulated(spec, n, N, "oneshot", torch.float32, "cuda", chunks)
    assert n % pipe.k == 0 and (n // pipe.k) % 1024 == 0
    for _ in range(2):  # reuse of the per-piece ops and events
        out.zero_()
        pipe(host, out)
        torch.cuda.synchronize()
        assert np.array_equal(out.numpy(), O.allreduce_oneshot(x64, O.scheme(spec)))
    dev = coll.SimulatedAllReduce(spec, n, N, "oneshot", torch.float32)([h.cuda() for h in host])
    assert torch.equal(dev.cpu(), out)
    assert pipe.h2d_bytes == N * n * 2 and pipe.d2h_bytes == n * 4


def test_host_pipeline_bf16_out_and_shape_checks(coll):
    n, N = 64 * 1024, 2
    x64 = [inputs.gauss_bf16(n, 90 + r) for r in range(N)]
    host = [_bf16(x).pin_memory() for x in x64]
    out = torch.empty(n, dtype=torch.bfloat16).pin_memory()
    pipe = coll.HostPipeline.simulated("fp4_e2m1:32:e8m0", n, N)
    pipe(host, out)
    torch.cuda.synchronize()
    ref = O.allreduce_oneshot(x64, O.scheme("fp4_e2m1:32:e8m0"))
    assert np.array_equal(out.float().numpy(), torch.from_numpy(ref).to(torch.bfloat16).float().numpy())
    from paper_2411_09510_b200.errors import ShapeMismatch

    with pytest.raises(ShapeMismatch):
        pipe(host[:1], out)


def test_flow_kernel_nonfinite_flag(coll):
    """The barrier-free fused kernel reports the first non-finite flat index."""
    n, N = 1 << 16, 2
    x64 = [inputs.gauss_bf16(n, 7 + r) for r in range(N)]
    x64[1] = x64[1].copy()
    x64[1][40000] = np.nan
    parts = [_bf16(x).cuda() for x in x64]
    sim = coll.SimulatedAllReduce("fp4_e2m1:32:e8m0", n, N, "oneshot", torch.float32)
    sim(parts)
    torch.cuda.synchronize()
    assert sim.fused and int(sim.flag.item()) == 40000


def test_host_pipeline_graph_cache_is_bounded(coll):
    n, N = 8 * 1024, 2
    x64 = [inputs.gauss_bf16(n, 300 + r) for r in range(N)]
    host = [_bf16(x).pin_memory() for x in x64]
    pipe = coll.HostPipeline.simulated("fp4_e2m1:32:e8m0", n, N, "oneshot", torch.float32,
                                       "cuda", 2)
    ref = O.allreduce_oneshot(x64, O.scheme("fp4_e2m1:32:e8m0"))
    outs = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(pipe.MAX_GRAPHS + 3)]
    for o in outs + outs[:2]:
        pipe(host, o)
    torch.cuda.synchronize()
    assert len(pipe._graphs) == pipe.MAX_GRAPHS
    for o in outs:
        assert np.array_equal(o.numpy(), ref)


def test_host_pipeline_weighted_pieces(coll):
    n, N = 64 * 1024, 2
    x64 = [inputs.gauss_bf16(n, 900 + r) for r in range(N)]
    host = [_bf16(x).pin_memory() for x in x64]
    out = torch.empty(n, dtype=torch.float32).pin_memory()
    pipe = coll.HostPipeline.simulated("fp4_e2m1:32:e8m0", n, N, "oneshot", torch.float32,
                                       "cuda", (1, 3, 3, 1))
    assert pipe.bounds == [0, 8192, 32768, 57344, 65536]
    pipe(host, out)
    torch.cuda.synchronize()
    assert np.array_equal(out.numpy(), O.allreduce_oneshot(x64, O.scheme("fp4_e2m1:32:e8m0")))
