"""GPU: the product collective at N > 1 ranks, on one device.

``CompressedAllReduce`` with the real ``NativeBackend`` runs its full NCCL
code path (K1 -> all_gather_into_tensor / all_to_all_single -> K3 -> K2)
for N = 2..8 ranks, each rank a host thread on its own stream, with
``LocalThreadGroup`` standing in for the process group (device copies in
rank order, torch.distributed signatures).  Every rank's result is checked
bit for bit against the pinned oracle (small and ragged sizes) or the
reference-generated digests (the 8B and 70B prefill shapes,
tests/golden/large.json), and all ranks must agree (mx/netbench.py:415-419).
``run_allgather_bench`` is checked against the reference's own reduced
tensors for the same seeds.
"""

import hashlib
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import mx_oracle as O  # noqa: E402
from tests.golden import inputs  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def large():
    with open(os.path.join(HERE, "golden", "large.json")) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2411_09510_b200 import _native

    return _native.load()


def run_ranks(parts_dev, spec, algo, out_dtype):
    """N ranks (threads) -> list of every rank's reduced tensor (host)."""
    from paper_2411_09510_b200.collective import CompressedAllReduce, LocalThreadGroup

    N = len(parts_dev)
    grp = LocalThreadGroup(N)

    def rank_fn(r):
        car = CompressedAllReduce(spec, parts_dev[r].numel(), algo=algo, out_dtype=out_dtype,
                                  comm=grp)
        assert car.world == N and car.rank == r
        out = car(parts_dev[r]).clone()
        out2 = car(parts_dev[r])  # a second call reuses the persistent buffers
        assert torch.equal(out, out2)
        car.check_finite()
        return out.float().cpu().numpy().ravel()

    return grp.run(rank_fn)


@pytest.mark.parametrize("N", [2, 3, 4, 8])
@pytest.mark.parametrize("algo", ["oneshot", "twoshot"])
def test_nccl_path_small_and_ragged(lib, N, algo):
    for spec, n in [("fp4_e2m1:32:e8m0", 8192), ("fp4_e2m1:32:e8m0", 5003),
                    ("fp5_e2m2:16:e5m0", 3000), ("int8:64:e8m0", 4096 + 64),
                    ("fp6_e3m2:32:e8m0", 1024 * N)]:
        x64 = [inputs.gauss_bf16(n, 900 + r) for r in range(N)]
        osch = O.scheme(spec)
        ref = (O.allreduce_oneshot if algo == "oneshot" else O.allreduce_twoshot)(x64, osch)
        for out_dt in (torch.float32, torch.bfloat16):
            parts = [torch.from_numpy(x).to("cuda", torch.bfloat16) for x in x64]
            outs = run_ranks(parts, spec, algo, out_dt)
            want = torch.from_numpy(ref).to(out_dt).float().numpy()
            for r, o in enumerate(outs):
                assert np.array_equal(o, want), (spec, n, N, algo, out_dt, r)


def test_nccl_path_matches_simulated_8b_shape(lib, large):
    """TP=2 one-shot at the 8B prefill shape against the reference digest,
    and TP=4 / TP=8 two-shot against the single-GPU simulation (itself
    pinned to the oracle), every rank bit-identical."""
    from paper_2411_09510_b200.collective import simulate_allreduce
    from paper_2411_09510_b200.synth import rank_partials

    shape = tuple(large["8b"]["shape"])
    host = rank_partials(shape, 8, seed=0)
    parts = [torch.from_numpy(p).to("cuda", torch.bfloat16) for p in host]
    outs = run_ranks(parts[:2], "fp4_e2m1:32:e8m0", "oneshot", torch.float32)
    for o in outs:
        assert sha(o.reshape(shape)) == large["8b"]["tp2_sum32"]
    outs = run_ranks(parts[:2], "fp4_e2m1:32:e8m0", "oneshot", torch.bfloat16)
    for o in outs:
        bits = torch.from_numpy(o).to(torch.bfloat16).view(torch.int16).numpy()
        assert sha(bits) == large["8b"]["tp2_sum_bf16"]
    for N in (4, 8):
        sim, _ = simulate_allreduce(parts[:N], "fp4_e2m1:32:e8m0", "twoshot", torch.float32)
        want = sim.float().cpu().numpy().ravel()
        outs = run_ranks(parts[:N], "fp4_e2m1:32:e8m0", "twoshot", torch.float32)
        for o in outs:
            assert np.array_equal(o, want), N


def test_70b_shape_parity(lib, large):
    """Llama-3.1-70B prefill partial [4096 x 8192]: K1 streams, the fused
    TP=2 step, and TP=8 one-shot both simulated and over the NCCL code path,
    against the reference's digests."""
    import paper_2411_09510_b200 as mx
    from paper_2411_09510_b200.collective import SimulatedAllReduce
    from paper_2411_09510_b200.synth import rank_partials

    g = large["70b"]
    shape = tuple(g["shape"])
    host = rank_partials(shape, 8, seed=0)
    assert [sha(p) for p in host] == g["input_sha"]
    parts = [torch.from_numpy(p).to("cuda", torch.bfloat16) for p in host]
    del host
    sch = mx.parse_scheme(large["scheme"])
    dct = mx.compress_tensor_device(parts[0], sch)
    assert sha(dct.scale.cpu().numpy()) == g["scale"]
    assert sha(dct.elements.cpu().numpy()) == g["elem"]
    n = parts[0].numel()
    for N in (2, 8):
        for out_dt, key in ((torch.float32, f"tp{N}_sum32"), (torch.bfloat16, f"tp{N}_sum_bf16")):
            op = SimulatedAllReduce(sch, n, N, "oneshot", out_dt, "cuda")
            assert op.fused
            out = op(parts[:N])
            got = out.view(torch.int16) if out_dt == torch.bfloat16 else out
            assert sha(got.cpu().numpy()) == g[key], (N, key)
            del op, out
    outs = run_ranks(parts, large["scheme"], "oneshot", torch.float32)
    for o in outs:
        assert sha(o.reshape(shape)) == g["tp8_sum32"]


@pytest.mark.parametrize("case", range(6))
def test_run_allgather_bench_vs_reference(lib, large, case):
    """run_allgather_bench: every worker ends with exactly the reduced tensor
    the reference's workers compute (sha1 as mx/netbench.py:335), and the
    BenchResult fields follow mx/netbench.py:461-472."""
    import math

    from paper_2411_09510_b200 import LinkModel, parse_scheme
    from paper_2411_09510_b200.netbench import _allgather_bench

    g = large["allgather"][case]
    sch = parse_scheme(g["scheme"]) if g["scheme"] else None
    res, digests = _allgather_bench(g["n_workers"], tuple(g["shape"]), sch,
                                    LinkModel(bandwidth=math.inf), repetitions=3,
                                    seed=g["seed"], compare_uncompressed=sch is not None)
    for rep in digests:
        assert rep == [g["sha1"]] * g["n_workers"]
    assert res.n_workers == g["n_workers"] and res.repetitions == 3
    assert res.wire_bytes_per_worker == g["wire_bytes_per_worker"]
    assert res.median_s > 0 and res.stddev_s >= 0
    if sch is not None:
        assert res.baseline_median_s is not None and res.speedup_vs_uncompressed > 0
    else:
        assert res.scheme == "none" and res.speedup_vs_uncompressed == 1.0


def test_run_allgather_bench_twoshot_and_throttle(lib):
    import math

    from paper_2411_09510_b200 import LinkModel, parse_scheme, run_allgather_bench

    sch = parse_scheme("fp4_e2m1:32:e8m0")
    r = run_allgather_bench(4, (128, 1024), sch, LinkModel(bandwidth=math.inf), repetitions=3,
                            algo="twoshot", compare_uncompressed=False)
    assert r.speedup_vs_uncompressed == 1.0 and r.baseline_median_s is None
    # a metered 1 GB/s link: the compressed payload ships ~3.8x faster
    link = LinkModel(bandwidth=1e9)
    r = run_allgather_bench(2, (256, 4096), sch, link, repetitions=3)
    assert r.median_s >= r.wire_bytes_per_worker / 1e9
    assert r.speedup_vs_uncompressed > 2.0


def test_calibrate_codec_throughput(lib):
    from paper_2411_09510_b200 import calibrate_codec_throughput, parse_scheme

    c, d = calibrate_codec_throughput(parse_scheme("fp4_e2m1:32:e8m0"), sample_sizes=(1 << 22,),
                                      repeats=5)
    assert c > 1e10 and d > 1e10  # values/s: far beyond the CPU reference's ~1e7
    c2, d2 = calibrate_codec_throughput(None, repeats=3, concurrency=2)
    assert c2 > 0 and d2 > 0


def test_blockwire_duck_type(lib, large):
    """BlockWire (mx/netbench.py:146-162) on the GPU codec reproduces the
    reference workers' reduction for the run_allgather_bench inputs."""
    from paper_2411_09510_b200 import parse_scheme
    from paper_2411_09510_b200.collective import BlockWire

    g = large["allgather"][1]  # 4 workers, fp4_e2m1:32:e8m0
    shape = tuple(g["shape"])
    rng = np.random.default_rng(g["seed"])
    tensors = [rng.standard_normal(shape).astype(np.float16) for _ in range(g["n_workers"])]
    wire = BlockWire(parse_scheme(g["scheme"]), shape)
    assert (g["n_workers"] - 1) * wire.payload_nbytes() == g["wire_bytes_per_worker"]
    enc = [wire.encode_with_reconstruction(t) for t in tensors]
    for rank in range(g["n_workers"]):
        red = np.zeros(shape, dtype=np.float32)
        for src in range(g["n_workers"]):
            red += enc[src][1] if src == rank else wire.decode(enc[src][0]).reshape(shape)
        assert hashlib.sha1(red.tobytes()).hexdigest() == g["sha1"]
