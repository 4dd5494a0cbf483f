"""The symmetric-memory fused collective on one GPU (world size 1): quantise
into the own shard slot, self flag exchange, pull-decode.  Bit-identical to
the unfused one-shot and the oracle, across repeated calls (epoch double
buffering).  Multi-GPU correctness follows from the same code path with
peer pointers; it cannot be exercised with a single device."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pg():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import torch.distributed as dist

    if not dist.is_initialized():
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("spec", ["fp4_e2m1:32:e8m0", "fp6_e2m3:64:e8m0", "int8:16:e8m0"])
def test_symm_world1_matches_oneshot(pg, spec):
    from oracle import mx_oracle as O
    from paper_2411_09510_b200.collective import SimulatedAllReduce, SymmetricAllReduce
    from tests.golden import inputs

    n = 1 << 20
    car = SymmetricAllReduce(spec, n, out_dtype=torch.float32)
    ref = SimulatedAllReduce(spec, n, 1, "oneshot", torch.float32, fused=False)
    for it in range(5):  # epochs 1..5: both slots, twice
        x64 = inputs.gauss_bf16(n, 3000 + it)
        x = torch.from_numpy(x64).to("cuda", torch.bfloat16)
        a = car(x).cpu().numpy().copy()
        b = ref([x]).cpu().numpy()
        assert np.array_equal(a, b), it
        assert np.array_equal(a, O.allreduce_oneshot([x64], O.scheme(spec))), it
    car.check_finite()
    car.check_status()


@pytest.mark.parametrize("spec", ["fp4_e2m1:32:e8m0", "int8:16:e8m0"])
def test_symm_twoshot_world1_real_symmetric_memory(pg, spec):
    """k_symm2_flow through torch symmetric memory (world size 1)."""
    from oracle import mx_oracle as O
    from paper_2411_09510_b200.collective import SymmetricAllReduce
    from tests.golden import inputs

    n = 1 << 18
    car = SymmetricAllReduce(spec, n, out_dtype=torch.float32, algo="twoshot")
    for it in range(4):
        x64 = inputs.gauss_bf16(n, 3300 + it)
        x = torch.from_numpy(x64).to("cuda", torch.bfloat16)
        a = car(x).cpu().numpy().copy()
        assert np.array_equal(a, O.allreduce_twoshot([x64], O.scheme(spec))), it
    car.check_status()


def test_row_parallel_linear_symm_algos(pg):
    """The TP hook with the one-kernel NVLink collectives equals the NCCL
    one-shot / two-shot hook bit for bit (world size 1)."""
    from paper_2411_09510_b200 import tp

    RowParallelLinear, _, _, _ = tp.make_module_classes()
    torch.manual_seed(0)
    x = torch.randn(2, 64, 512, device="cuda", dtype=torch.bfloat16)
    for nccl, symm in (("oneshot", "symm"), ("twoshot", "symm2")):
        a = RowParallelLinear(512, 256, scheme="fp4_e2m1:32:e8m0", algo=nccl)
        b = RowParallelLinear(512, 256, scheme="fp4_e2m1:32:e8m0", algo=symm)
        b.weight.data.copy_(a.weight.data)
        for _ in range(3):
            assert torch.equal(a(x), b(x)), (nccl, symm)
