"""Multi-process (gloo, world_size 2, 3 and 4) test of the collective's
orchestration on CPU: shard layout, chunking, all_to_all / all_gather order
and the rank-order reduction, with the oracle standing in for the kernels."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, specs, n, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle import mx_oracle as O
        from paper_2411_09510_b200.collective import CompressedAllReduce
        from paper_2411_09510_b200.formats import parse_scheme
        from tests.golden import inputs
        from tests.oracle_backend import OracleBackend

        x64 = [inputs.gauss_bf16(n, 500 + r) for r in range(world)]
        for spec in specs:
            sch = parse_scheme(spec, extensions=True)
            for algo in ("oneshot", "twoshot"):
                car = CompressedAllReduce(sch, n, algo=algo, out_dtype=torch.float32,
                                          device="cpu", backend=OracleBackend(sch))
                out = car(torch.from_numpy(x64[rank]).float()).numpy().copy()
                ref = (O.allreduce_oneshot if algo == "oneshot" else O.allreduce_twoshot)(
                    x64, O.scheme(spec))
                assert np.array_equal(out, ref), (spec, algo, rank)
                # every rank ends bit-identical (mx/netbench.py:415-419)
                allv = [torch.zeros(n) for _ in range(world)]
                dist.all_gather(allv, torch.from_numpy(out))
                assert all(torch.equal(allv[0], a) for a in allv)
                if algo == "oneshot":
                    assert car.wire_bytes_per_rank == (world - 1) * car.plan.shard_bytes
                # the residual-fused form: out = h + all_reduce(x), in place
                h = torch.from_numpy(inputs.gauss_bf16(n, 900 + rank)).float()
                want = h + torch.from_numpy(ref)
                got = car(torch.from_numpy(x64[rank]).float(), out=h, residual=h)
                assert got.data_ptr() == h.data_ptr() and torch.equal(got, want), (spec, algo)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback

        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("world", [2, 3, 4])
def test_collective_orchestration_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    specs = ["fp4_e2m1:32:e8m0", "fp5_e2m2:16:e5m0"]
    procs = [ctx.Process(target=_worker, args=(r, world, port, specs, 5003, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    bad = [r for r in res if r[1] != "ok"]
    assert not bad, bad[0][1]
