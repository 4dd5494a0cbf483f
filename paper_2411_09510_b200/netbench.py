"""The reference's collective benchmark and cost model, on the GPU path.

Mirrors ``mxcomm.netbench`` (mx/netbench.py) name for name:

* :class:`LinkModel`, :func:`predict_comm_time`, :func:`predicted_speedup`
  -- the analytic full-mesh model (mx/netbench.py:57-72, 480-516), same
  arithmetic.
* :class:`BenchResult` / :func:`run_allgather_bench` -- the measured
  compress -> exchange -> decompress -> fp32 rank-order reduce collective
  (mx/netbench.py:76-84, 307-472).  The reference runs N worker threads over
  in-process mailboxes or loopback TCP with a token bucket per worker; here
  each worker owns a :class:`~.collective.CompressedAllReduce` (K1 -> all-
  gather -> K2, the product path) and the exchange is either
  ``transport="memory"``: N threads sharing this GPU through
  :class:`~.collective.LocalThreadGroup` (device copies), or
  ``transport="nccl"``: one worker per process of the initialised
  torch.distributed group (NCCL over NVLink).  Inputs are the reference's
  (``default_rng(seed).standard_normal(shape).astype(float16)`` per worker),
  one untimed warm-up repetition precedes the timed ones, every worker's
  reduced fp32 tensor is hashed after every repetition and any disagreement
  raises :class:`ResultMismatch` (mx/netbench.py:415-419).
* :func:`calibrate_codec_throughput` -- values/s of compress-with-
  reconstruction and decode-plus-accumulate (mx/netbench.py:528-578), timed
  with CUDA events on the device codec.

A finite ``link.bandwidth`` meters each worker's sends the way the
reference's token bucket does -- (N-1) x (latency + payload / bandwidth) of
host-side wait per repetition (mx/netbench.py:296-304) -- so the modelled
crossover can be reproduced; ``bandwidth=math.inf`` times the real link.
"""

from __future__ import annotations

import hashlib
import math
import statistics
import threading
import time
from dataclasses import dataclass

import numpy as np

from .errors import MinimumDegreeTwo, ResultMismatch, TransportFailure

UNCOMPRESSED_VALUE_BYTES = 2
TRANSPORTS = ("memory", "nccl")


@dataclass(frozen=True)
class LinkModel:
    """A point-to-point link plus the codec rates at its endpoints
    (mx/netbench.py:57-72)."""

    bandwidth: float  # bytes per second
    latency: float = 0.0  # seconds per message
    compress_throughput: float = math.inf  # values per second
    decompress_throughput: float = math.inf  # values per second

    def __post_init__(self):
        if not self.bandwidth > 0:
            raise ValueError("bandwidth must be positive")
        if self.latency < 0:
            raise ValueError("latency cannot be negative")
        if not (self.compress_throughput > 0 and self.decompress_throughput > 0):
            raise ValueError("codec throughputs must be positive")


@dataclass(frozen=True)
class BenchResult:
    """mx/netbench.py:76-84"""

    scheme: str
    n_workers: int
    repetitions: int
    median_s: float
    stddev_s: float
    wire_bytes_per_worker: int
    speedup_vs_uncompressed: float
    baseline_median_s: float | None = None


def predict_comm_time(tensor_bytes: int, scheme, n_workers: int, link: LinkModel) -> float:
    """Full-mesh model (mx/netbench.py:480-505): uncompressed
    ``(N-1)(latency + bytes/bw)``; compressed ships the MXC1 container and
    adds one compression and N-1 decompression passes."""
    from .codec import serialized_nbytes

    if n_workers < 2:
        raise MinimumDegreeTwo(f"need at least 2 workers, got {n_workers}")
    peers = n_workers - 1
    base = peers * link.latency
    if scheme is None:
        return base + peers * tensor_bytes / link.bandwidth
    values = tensor_bytes // UNCOMPRESSED_VALUE_BYTES
    wire = serialized_nbytes(scheme, (values,))
    return (base + peers * wire / link.bandwidth + values / link.compress_throughput
            + peers * values / link.decompress_throughput)


def predicted_speedup(tensor_bytes: int, scheme, n_workers: int, link: LinkModel) -> float:
    """mx/netbench.py:508-516"""
    return (predict_comm_time(tensor_bytes, None, n_workers, link)
            / predict_comm_time(tensor_bytes, scheme, n_workers, link))


# ---------------------------------------------------------------------------
# the measured collective
# ---------------------------------------------------------------------------


class _RawAllGather:
    """scheme=None: ship the 16-bit tensor unchanged, fp32 rank-order sum
    (mx/netbench.py:127-143) -- the uncompressed comparison arm."""

    name = "none"

    def __init__(self, n, comm, world, rank, device):
        import torch

        self.n, self.comm, self.world, self.rank = n, comm, world, rank
        self.gathered = torch.empty(world * n, dtype=torch.float16, device=device)
        self.out = torch.empty(n, dtype=torch.float32, device=device)

    def __call__(self, x):
        mine = self.gathered[self.rank * self.n:(self.rank + 1) * self.n]
        mine.copy_(x.reshape(-1))
        self.comm.all_gather_into_tensor(self.gathered, mine)
        self.out.zero_()  # +0.0 start, rank order (mx/netbench.py:332-334)
        for r in range(self.world):
            self.out += self.gathered[r * self.n:(r + 1) * self.n].float()
        return self.out


def _make_op(scheme, n, comm, world, rank, device, algo):
    import torch

    from .collective import CompressedAllReduce

    if scheme is None:
        return _RawAllGather(n, comm, world, rank, device)
    return CompressedAllReduce(scheme, n, algo=algo, out_dtype=torch.float32, device=device,
                               world_size=world, rank=rank, comm=comm)


def _send_delay(link: LinkModel, payload: int, n_workers: int) -> float:
    if not math.isfinite(link.bandwidth) and link.latency == 0:
        return 0.0
    per = link.latency + (payload / link.bandwidth if math.isfinite(link.bandwidth) else 0.0)
    return (n_workers - 1) * per


def _payload_nbytes(scheme, shape) -> int:
    from .codec import serialized_nbytes

    if scheme is None:
        return int(np.prod(shape, dtype=np.int64)) * UNCOMPRESSED_VALUE_BYTES
    return serialized_nbytes(scheme, tuple(shape))


def _digest(out) -> str:
    return hashlib.sha1(out.detach().cpu().numpy().tobytes()).hexdigest()


def _run_memory(n_workers, tensors, scheme, link, repetitions, algo, device):
    """N worker threads on this GPU; the orchestrator times each repetition
    between two barriers, as mx/netbench.py:392-399 does."""
    import torch

    from .collective import LocalThreadGroup

    shape = tuple(tensors[0].shape)
    n = int(np.prod(shape, dtype=np.int64))
    payload = _payload_nbytes(scheme, shape)
    delay = _send_delay(link, payload, n_workers)
    grp = LocalThreadGroup(n_workers, device)
    total = repetitions + 1  # the first repetition is an untimed warm-up
    gate = threading.Barrier(n_workers + 1)
    digests = [[None] * n_workers for _ in range(total)]
    failures = []

    def worker(r):
        try:
            torch.cuda.set_device(grp.device)
            grp.bind(r)
            st = torch.cuda.Stream(grp.device)
            with torch.cuda.stream(st):
                x = torch.from_numpy(tensors[r]).to(grp.device)
                op = _make_op(scheme, n, grp, n_workers, r, grp.device, algo)
                st.synchronize()
                for rep in range(total):
                    gate.wait()
                    if delay:
                        time.sleep(delay)  # metered sends (token bucket)
                    out = op(x)
                    st.synchronize()
                    gate.wait()
                    digests[rep][r] = _digest(out)
        except BaseException as exc:  # noqa: BLE001  (propagated below)
            failures.append((r, exc))
            gate.abort()
            grp.abort()

    threads = [threading.Thread(target=worker, args=(r,), daemon=True)
               for r in range(n_workers)]
    for t in threads:
        t.start()
    times = []
    try:
        for _ in range(total):
            gate.wait()
            t0 = time.perf_counter()
            gate.wait()
            times.append(time.perf_counter() - t0)
    except threading.BrokenBarrierError:
        pass
    for t in threads:
        t.join(timeout=60.0)
    if failures:
        r, exc = next(((r, e) for r, e in failures
                       if not isinstance(e, threading.BrokenBarrierError)), failures[0])
        raise TransportFailure(f"worker {r} failed: {exc}") from exc
    return times[1:], digests


def _run_nccl(n_workers, tensors, scheme, link, repetitions, algo, device):
    """One worker per process of the torch.distributed group."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized():
        raise TransportFailure("transport 'nccl' needs an initialised process group")
    world, rank = dist.get_world_size(), dist.get_rank()
    if world != n_workers:
        raise TransportFailure(f"n_workers {n_workers} != process group size {world}")
    shape = tuple(tensors[0].shape)
    n = int(np.prod(shape, dtype=np.int64))
    delay = _send_delay(link, _payload_nbytes(scheme, shape), n_workers)
    dev = torch.device(device) if device is not None else torch.device(
        "cuda", torch.cuda.current_device())
    x = torch.from_numpy(tensors[rank]).to(dev)
    op = _make_op(scheme, n, dist, world, rank, dev, algo)
    times, mine = [], []
    for _ in range(repetitions + 1):
        dist.barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        if delay:
            time.sleep(delay)
        out = op(x)
        torch.cuda.synchronize(dev)
        dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)  # the slowest worker ends the collective
        times.append(float(dt.item()))
        mine.append(_digest(out))
    allg = [None] * world
    dist.all_gather_object(allg, mine)
    digests = [[allg[r][rep] for r in range(world)] for rep in range(repetitions + 1)]
    return times[1:], digests


def _run_configuration(n_workers, tensors, scheme, link, repetitions, transport, algo, device):
    if transport == "memory":
        timed, digests = _run_memory(n_workers, tensors, scheme, link, repetitions, algo, device)
    elif transport == "nccl":
        timed, digests = _run_nccl(n_workers, tensors, scheme, link, repetitions, algo, device)
    else:
        raise ValueError(f"unknown transport {transport!r}")
    for rep, d in enumerate(digests):
        if len(set(d)) != 1:
            raise ResultMismatch(f"repetition {rep}: workers disagree on the reduced tensor")
    name = "none" if scheme is None else scheme.name
    return timed, (n_workers - 1) * _payload_nbytes(scheme, tensors[0].shape), name, digests


def run_allgather_bench(n_workers: int, shape, scheme, link: LinkModel, repetitions: int = 5,
                        transport: str = "memory", seed: int = 0,
                        compare_uncompressed: bool = True, algo: str = "oneshot",
                        device=None) -> BenchResult:
    """Measure the compress/exchange/decompress/reduce collective
    (mx/netbench.py:424-472) on the GPU path; see the module docstring.
    ``algo`` ("oneshot" as the reference, or "twoshot") picks the
    compressed exchange."""
    res, _ = _allgather_bench(n_workers, shape, scheme, link, repetitions, transport, seed,
                              compare_uncompressed, algo, device)
    return res


def _allgather_bench(n_workers, shape, scheme, link, repetitions=5, transport="memory", seed=0,
                     compare_uncompressed=True, algo="oneshot", device=None):
    """run_allgather_bench plus the per-repetition digests (tests)."""
    from . import _native

    if n_workers < 2:
        raise MinimumDegreeTwo(f"need at least 2 workers, got {n_workers}")
    if repetitions < 3:
        raise ValueError("need at least 3 repetitions for a stable median")
    if transport not in TRANSPORTS:
        raise ValueError(f"unknown transport {transport!r}")
    _native.require_cuda()
    shape = tuple(int(d) for d in shape)
    rng = np.random.default_rng(seed)
    tensors = [rng.standard_normal(shape).astype(np.float16) for _ in range(n_workers)]
    timed, wire_bytes, name, digests = _run_configuration(
        n_workers, tensors, scheme, link, repetitions, transport, algo, device)
    median = statistics.median(timed)
    baseline_median, speedup = None, 1.0
    if scheme is not None and compare_uncompressed:
        base, _, _, _ = _run_configuration(n_workers, tensors, None, link, repetitions,
                                           transport, algo, device)
        baseline_median = statistics.median(base)
        speedup = baseline_median / median
    return BenchResult(scheme=name, n_workers=n_workers, repetitions=repetitions,
                       median_s=median, stddev_s=statistics.stdev(timed),
                       wire_bytes_per_worker=wire_bytes, speedup_vs_uncompressed=speedup,
                       baseline_median_s=baseline_median), digests


# ---------------------------------------------------------------------------
# codec throughput calibration
# ---------------------------------------------------------------------------


def calibrate_codec_throughput(scheme, sample_sizes=(1 << 22,), repeats: int = 5,
                               concurrency: int = 1, seed: int = 0):
    """(compress, decompress) throughput in values/second
    (mx/netbench.py:528-578): compression WITH local reconstruction (K1,
    then the own shard decoded to fp32) and decode-plus-accumulate (K2 of one
    shard into fp32, added to an accumulator), each the median of
    ``repeats`` CUDA-event-timed calls on fp16 data.  ``concurrency`` > 1
    runs that many measuring threads at once on their own streams (shared-
    GPU contention, as the reference's thread pool)."""
    import torch

    from . import _native

    if repeats < 1:
        raise ValueError("repeats must be at least 1")
    _native.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    rng = np.random.default_rng(seed)

    def measure(size):
        data = torch.from_numpy(rng.standard_normal(size).astype(np.float16)).to(dev)
        # the worker threads use their own non-blocking streams
        torch.cuda.current_stream(dev).synchronize()

        def thread_rates():
            torch.cuda.set_device(dev)
            st = torch.cuda.Stream(dev)
            with torch.cuda.stream(st):
                acc = torch.zeros(size, dtype=torch.float32, device=dev)
                if scheme is None:
                    own = torch.empty(size, dtype=torch.float32, device=dev)

                    def comp():
                        own.copy_(data)

                    def decomp():
                        acc.add_(data.float())
                else:
                    from .collective import NativeBackend

                    be = NativeBackend(scheme)
                    _, _, S = be.layout(size)
                    shard = torch.empty(S, dtype=torch.uint8, device=dev)
                    ws = torch.empty(max(16, be.workspace(size)), dtype=torch.uint8, device=dev)
                    flag = torch.empty(1, dtype=torch.int64, device=dev)
                    be.reset_flag(flag)
                    own = torch.empty(size, dtype=torch.float32, device=dev)
                    dec = torch.empty(size, dtype=torch.float32, device=dev)

                    def comp():
                        be.quantize_into(data, shard, ws, flag)
                        be.dequant_sum(shard, S, 1, size, size, 0, own)

                    def decomp():
                        be.dequant_sum(shard, S, 1, size, size, 0, dec)
                        acc.add_(dec)

                    comp()

                def median_s(op):
                    ts = []
                    for _ in range(repeats):
                        e0 = torch.cuda.Event(enable_timing=True)
                        e1 = torch.cuda.Event(enable_timing=True)
                        e0.record(st)
                        op()
                        e1.record(st)
                        e1.synchronize()
                        ts.append(e0.elapsed_time(e1) * 1e-3)
                    return max(statistics.median(ts), 1e-9)

                comp()
                decomp()
                return size / median_s(comp), size / median_s(decomp)

        if concurrency == 1:
            return thread_rates()
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(max_workers=concurrency) as pool:
            rates = list(pool.map(lambda _: thread_rates(), range(concurrency)))
        return (statistics.median(r[0] for r in rates), statistics.median(r[1] for r in rates))

    per = [measure(int(s)) for s in sample_sizes]
    return (statistics.median(r[0] for r in per), statistics.median(r[1] for r in per))
