#!/usr/bin/env python
"""Benchmark of the compressed TP all-reduce (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One *step* = one compressed all-reduce of the Llama-3.1-8B prefill
row-parallel partial sum [2048 x 4096] bf16 (MXFP4 block 32, E8M0 scales,
one-shot): quantise (K1) -> exchange -> unpack/dequantise/fp32 rank-order
sum -> bf16 (K2).

* N = 1 (default): BASELINE.json configs[0] on one B200 -- "simulated TP=2":
  two rank partials are quantised into the gathered buffer exactly as the
  NCCL all-gather would leave it, then K2 reduces both shards.
* N > 1 (torchrun, one rank per GPU): real TP=N over NCCL (NVLink 5), one
  partial per GPU (weak scaling), plus the uncompressed bf16 NCCL
  all-reduce on the same tensor for the speed-up.

``value`` = bf16 bytes of partial sums reduced per second over the whole
job (ranks x 2n bytes / step time), device-timed with CUDA events over
exactly K CUDA-graph replays, inputs resident in HBM and rotated over buffer
sets larger than L2.  ``e2e`` is the same metric through the public API with
pinned host buffers (H2D of the partials and D2H of the result inside the
timed region).  ``roofline`` is the dominant kernel (K1) against the
measured HBM copy bandwidth.  ``cpu_baseline`` is the CPU oracle (a numpy
restatement of the reference codec; the reference itself is Python and does
not travel to the GPU box) on the box's host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
UNIT = "GB/s"
L2_BYTES = 126 * 2 ** 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--scheme", default="fp4_e2m1:32:e8m0")
    ap.add_argument("--algo", choices=["auto", "oneshot", "twoshot"], default="auto",
                    help="auto: one-shot up to TP=2, two-shot from TP=4 (DESIGN.md (e))")
    ap.add_argument("--shape", default="2048,4096")
    ap.add_argument("--sim-ranks", type=int, default=2, help="simulated TP degree at N=1")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-pieces", default="1,3,3,1",
                    help="HostPipeline piece weights (or one integer: equal pieces)")
    ap.add_argument("--profile", action="store_true",
                    help="ncu mode: a few eager launches, no timing, no JSON")
    return ap.parse_args()


def peaks():
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)
# ---------------------------------------------------------------------------


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        loaded = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm), "samples_loaded": len(loaded)}


# ---------------------------------------------------------------------------
# CPU baselines (the oracle restatement of the reference codec)
# ---------------------------------------------------------------------------


_POOL = {}


def _pool(threads):
    from concurrent.futures import ThreadPoolExecutor

    if threads not in _POOL:  # one pool per process: no per-step thread start-up
        _POOL[threads] = ThreadPoolExecutor(threads)
    return _POOL[threads]


def cpu_oracle_step(partials64, spec, threads):
    """One simulated-TP compress+reduce cycle of the reference semantics
    (mx/netbench.py:323-334) on host cores, blocks split over threads."""
    from oracle import mx_oracle as O

    sch = O.scheme(spec)
    n = partials64[0].size
    unit = 8 * sch.block
    per = -(-n // threads)
    per = -(-per // unit) * unit
    sls = [slice(i * per, min(n, (i + 1) * per)) for i in range(threads) if i * per < n]

    def work(sl):
        return O.allreduce_oneshot([p.reshape(-1)[sl] for p in partials64], sch)

    if threads == 1 or len(sls) == 1:
        return work(slice(0, n))
    return np.concatenate(list(_pool(threads).map(work, sls)))


def cpu_baseline(spec, shape, nranks, budget_s=10.0):
    from paper_2411_09510_b200.synth import rank_partials

    threads = os.cpu_count() or 1
    parts = [p.astype(np.float64) for p in rank_partials(shape, nranks, seed=0)]
    n = parts[0].size
    times = []
    t_all = time.perf_counter()
    while True:
        t = time.perf_counter()
        cpu_oracle_step(parts, spec, threads)
        times.append(time.perf_counter() - t)
        if len(times) >= 2 and time.perf_counter() - t_all > budget_s:
            break
    med = statistics.median(times)
    return {"value": round(nranks * 2 * n / med / 1e9, 4), "unit": UNIT, "cores": threads,
            "kind": "port",
            "sample": f"{len(times)} full steps of simulated TP={nranks} on {list(shape)} "
                      f"({spec}); median {med * 1e3:.1f} ms/step; oracle/mx_oracle.py "
                      f"(numpy restatement of mx/codec.py + mx/netbench.py:332-334), "
                      f"blocks split over {threads} threads"}


def run_reference(args, shape, rank, world):
    """--impl reference: the CPU reference path (oracle port) on host cores,
    rank 0 only; each step a bounded row-sample of the same workload."""
    if rank != 0:
        return
    from paper_2411_09510_b200.synth import rank_partials

    T, H = shape
    nranks = args.sim_ranks if world == 1 else world
    threads = os.cpu_count() or 1
    # calibrate: seconds per row for the full cycle (pool warm, 128 rows)
    cal_rows = 128
    cal = [p.astype(np.float64) for p in rank_partials((cal_rows, H), nranks, seed=0)]
    cpu_oracle_step(cal, args.scheme, threads)
    t = time.perf_counter()
    cpu_oracle_step(cal, args.scheme, threads)
    per_row = (time.perf_counter() - t) / cal_rows
    # each step: as many rows as a ~120 s run allows (at least 8)
    budget = 120.0
    rows = int(min(T, budget / max(1, args.steps + args.warmup) / max(per_row, 1e-9)))
    rows = min(T, max(8, (rows // 8) * 8))
    parts = [p.astype(np.float64) for p in rank_partials((rows, H), nranks, seed=0)]
    for _ in range(args.warmup):
        cpu_oracle_step(parts, args.scheme, threads)
    t = time.perf_counter()
    for _ in range(args.steps):
        cpu_oracle_step(parts, args.scheme, threads)
    el = time.perf_counter() - t
    ms = el / args.steps * 1e3
    value = nranks * 2 * rows * H / (el / args.steps) / 1e9
    sample = (f"{rows} of {T} rows x {H} per step, {nranks} rank partials, {args.scheme}; "
              f"oracle/mx_oracle.py (numpy restatement of the reference codec) on "
              f"{threads} host threads")
    line = {"metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (gaussian_with_outliers, mx/synth.py)",
            "impl": "reference",
            "config": config_dict(args, shape, world),
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": threads,
                             "kind": "port", "sample": sample},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_dict(args, shape, world):
    sim = world == 1
    return {"workload": (f"Llama-3.1-8B prefill row-parallel all-reduce [{shape[0]}x{shape[1]}] "
                         f"bf16, {args.scheme}, {args.algo}, "
                         + (f"simulated TP={args.sim_ranks} on 1 GPU (BASELINE configs[0])"
                            if sim else f"TP={world} over NCCL (BASELINE configs[1])")),
            "scheme": args.scheme, "algo": args.algo, "tp": args.sim_ranks if sim else world,
            "ranks_per_gpu": args.sim_ranks if sim else 1, "seq_len": shape[0],
            "hidden": shape[1],
            "l2": "inputs rotated over buffer sets totalling > 126 MB L2"}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------


def time_graph_replays(torch, graphs, k):
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for i in range(k):
        graphs[i % len(graphs)].replay()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)  # ms


def time_steps(torch, g_all, graphs, k):
    """Exactly k steps: k // R replays of the graph holding all R buffer
    sets' steps back to back, then k % R single-step replays (a multi-step
    graph amortises the graph-launch overhead the way a captured prefill
    forward does; every step still runs in full)."""
    R = len(graphs)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(k // R):
        g_all.replay()
    for i in range(k % R):
        graphs[i].replay()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)  # ms


def capture(torch, fn):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()  # warm (first-call allocations happen outside the graph)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        fn()
    torch.cuda.synchronize()
    return g


def load_traffic(kernel_key):
    """dram bytes per launch from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        return json.load(open(path)).get(kernel_key)
    except Exception:
        return None


def run_ours(args, shape, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2411_09510_b200 import _native
    from paper_2411_09510_b200.collective import (CompressedAllReduce, SimulatedAllReduce,
                                                  twoshot_chunk_values)
    from paper_2411_09510_b200.formats import parse_scheme
    from paper_2411_09510_b200.synth import rank_partials

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    _native.load()
    sch = parse_scheme(args.scheme, extensions=True)
    T, H = shape
    n = T * H
    sim = world == 1
    nranks = args.sim_ranks if sim else world
    so, eo, S = _native.shard_layout(n, sch.to_c())
    sb, eb = _native.stream_nbytes(n, sch.to_c())
    # buffer sets: one pass over them moves > 3x L2, so every step and every
    # timed kernel launch reads data that is not L2-resident
    per_set = (nranks if sim else 1) * 2 * n + (nranks * S) + 2 * n
    R = max(3, -(-3 * L2_BYTES // per_set))
    mine = list(range(nranks)) if sim else [rank]  # the partials this GPU owns
    host_parts = {r: rank_partials(shape, 1, seed=r)[0] for r in mine}  # seed = rank
    base = [torch.from_numpy(host_parts[r]).to(dev, torch.bfloat16) for r in mine]
    sets = []
    for s in range(R):
        # distinct data per set: row roll + sign flip keep the statistics
        parts = [(b.roll(s * 7, 0) * (-1) ** s).contiguous() for b in base]
        if sim:
            op = SimulatedAllReduce(sch, n, nranks, args.algo, torch.bfloat16, dev)
        else:
            op = CompressedAllReduce(sch, n, algo=args.algo, out_dtype=torch.bfloat16, device=dev)
        sets.append((parts, op))

    def step_fn(i):
        parts, op = sets[i]
        return (lambda: op(parts)) if sim else (lambda: op(parts[0]))

    if args.profile:  # ncu: eager launches only
        for i in range(3):
            step_fn(i % R)()
        torch.cuda.synchronize()
        return

    graphs = [capture(torch, step_fn(i)) for i in range(R)]
    steps_all = [step_fn(i) for i in range(R)]
    g_all = capture(torch, lambda: [f() for f in steps_all])
    fused = sim and getattr(sets[0][1], "fused", False)
    if fused:  # one persistent kernel per step (quantise, grid barrier, dequant-sum)
        launches_per_step = 1
    elif args.algo == "oneshot":  # K1 x local partials + K2
        launches_per_step = (nranks if sim else 1) + 1
    else:  # two-shot: K1 x ranks, K3 x owned chunks, K2
        launches_per_step = (nranks if sim else 1) + (nranks if sim else 1) + 1

    # warm-up (>= W replays and >= 0.3 s so clocks settle), timed region.
    # The replay count is agreed across ranks (each replay may hold NCCL
    # collectives, so every rank must run exactly as many).
    with ClockSampler(local_rank) as clk:
        t = time.perf_counter()
        for i in range(args.warmup):
            graphs[i % R].replay()
        torch.cuda.synchronize()
        el = time.perf_counter() - t
        extra = 0
        if el < 0.3:
            extra = int(min(1e6, (0.3 - el) / max(el / max(1, args.warmup), 1e-6))) + 1
        if world > 1:
            te = torch.tensor([extra], device=dev, dtype=torch.int64)
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
            extra = int(te.item())
        for i in range(extra):
            graphs[i % R].replay()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ms_total = time_steps(torch, g_all, graphs, args.steps)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
    clocks = clk.summary()
    ms_local = ms_total / args.steps
    ms_step = ms_local
    if world > 1:
        tt = torch.tensor([ms_local], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_step = float(tt.item())
    value = nranks * 2 * n / (ms_step * 1e-3) / 1e9

    # ---- per-kernel device times (roofline), graphs of back-to-back launches
    kernels = {}
    if sim and args.algo == "oneshot":
        # one graph = one launch per buffer set (R distinct inputs > 3x L2)
        def q_all():
            for parts, op in sets:
                op.be.quantize_into(parts[0].reshape(-1), op.gathered[0:S], op.ws, op.flag)

        def d_all():
            for parts, op in sets:
                op.reduce()

        for name, fn, bytes_per in (("k_quant", q_all, 2 * n + sb + eb),
                                    ("k_dqsum", d_all, nranks * (sb + eb) + 2 * n)):
            g = capture(torch, fn)
            for _ in range(3):
                g.replay()
            reps = max(4, min(100, args.steps // 20))
            ms = time_graph_replays(torch, [g], reps) / (reps * R)
            kernels[name] = {"us": round(ms * 1e3, 3), "bytes": bytes_per,
                             "gbs": round(bytes_per / (ms * 1e-3) / 1e9, 1),
                             "launches_timed": reps * R}
    if not sim and args.algo == "oneshot":
        # N>1: this rank's K1 and its K2 over the N gathered shards, timed on
        # the rank's own buffers (local launches only, no collective)
        try:
            def q_all():
                for parts, op in sets:
                    S_ = op.plan.shard_bytes
                    op.backend.quantize_into(parts[0].reshape(-1),
                                             op.gathered[rank * S_:(rank + 1) * S_], op.ws,
                                             op.flag)

            def d_all():
                for parts, op in sets:
                    S_ = op.plan.shard_bytes
                    op.backend.dequant_sum(op.gathered, S_, world, n, n, 0, op.out)

            for name, fn, bytes_per in (("k_quant", q_all, 2 * n + sb + eb),
                                        ("k_dqsum", d_all, world * (sb + eb) + 2 * n)):
                g = capture(torch, fn)
                for _ in range(3):
                    g.replay()
                reps = max(4, min(100, args.steps // 20))
                ms = time_graph_replays(torch, [g], reps) / (reps * R)
                kernels[name] = {"us": round(ms * 1e3, 3), "bytes": bytes_per,
                                 "gbs": round(bytes_per / (ms * 1e-3) / 1e9, 1),
                                 "launches_timed": reps * R}
        except Exception as exc:  # noqa: BLE001  (reported, never fatal)
            kernels = {"error": f"{type(exc).__name__}: {exc}"[:200]}
    peak, peak_kind = peaks()
    roof = None
    if not sim and "k_dqsum" in kernels:
        kd = kernels["k_dqsum"]
        roof = {"bound": "hbm",
                "kernel": f"k_dqsum_lean<bf16,B={sch.block_size},{sch.element.name}> "
                          f"(K2: {world} gathered shards -> bf16, this rank)",
                "achieved": kd["gbs"], "peak": peak, "unit": "GB/s",
                "frac": round(kd["gbs"] / peak, 4), "traffic": None,
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind}, burst copy)",
                "algorithmic_bytes_per_launch": kd["bytes"], "launch_us": kd["us"],
                "share_of_step": round(kd["us"] / (ms_step * 1e3), 3),
                "other_kernels": {k: v for k, v in kernels.items() if k != "k_dqsum"},
                "note": "rank 0's device time; the NCCL all-gather is the rest of the step"}
    elif fused and "k_quant" in kernels:
        # the step IS one kernel (k_fused_flow): it must read the N partials
        # from HBM, write the N shards into the gather buffer (the bytes an
        # all-gather delivers) and write the bf16 sum.  Each warp reads its
        # shard slices straight back (L2 hits by construction), so the
        # read-back is reported separately and NOT counted as HBM traffic.
        fb = nranks * 2 * n + nranks * (sb + eb) + 2 * n
        ach = round(fb / (ms_step * 1e-3) / 1e9, 1)
        tr = load_traffic(f"k_fused_flow|{args.scheme}|{T}x{H}|bf16|{nranks}ranks")
        traffic = tr.get("per_launch_bytes") if isinstance(tr, dict) else tr
        roof = {"bound": "hbm",
                "kernel": f"k_fused_flow<bf16,B={sch.block_size},{sch.element.name}> "
                          f"(quantise {nranks} partials -> gather buffer -> read back, "
                          f"dequant-sum; one launch, no grid barrier)",
                "achieved": ach, "peak": peak, "unit": "GB/s", "frac": round(ach / peak, 4),
                "traffic": traffic,
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind}, burst copy)",
                "algorithmic_bytes_per_launch": fb,
                "algorithmic_bytes_note": "N*2n partial reads + N*S shard writes + 2n output; "
                                          f"+{nranks * (sb + eb)} B shard read-back from L2 "
                                          "not counted",
                "launch_us": round(ms_step * 1e3, 3),
                "share_of_step": 1.0,
                "unfused_kernels": kernels}
    elif "k_quant" in kernels:
        # dominant kernel: K1 runs nranks times per step
        kq = kernels["k_quant"]
        ach = kq["gbs"]
        tr = load_traffic(f"k_quant|{args.scheme}|{T}x{H}|bf16")
        traffic = tr.get("per_launch_bytes") if isinstance(tr, dict) else tr
        roof = {"bound": "hbm", "kernel": f"k_quant<bf16,B={sch.block_size},{sch.element.name}> (K1 quantise+pack)",
                "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "traffic": traffic,
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind}, burst copy)",
                "algorithmic_bytes_per_launch": kq["bytes"],
                "launch_us": kq["us"],
                "share_of_step": round(nranks * kq["us"] / (ms_step * 1e3), 3),
                "other_kernels": {k: v for k, v in kernels.items() if k != "k_quant"}}

    # ---- simulated TP=4 and TP=8 on this GPU (N=1): the fused one-kernel
    # step with 4 / 8 rank partials (inputs rotated > 3x L2), informational
    sim_more = None
    if sim and args.algo == "oneshot" and args.sim_ranks == 2:
        sim_more = {}
        try:
            for N_ in (4, 8):
                per = N_ * 2 * n + N_ * S + 2 * n
                R_ = max(2, -(-3 * L2_BYTES // per))
                ps = [[(base[r % len(base)].roll(7 * (i + r), 0) * (-1) ** (i + r)).contiguous()
                       for r in range(N_)] for i in range(R_)]
                ops = [SimulatedAllReduce(sch, n, N_, "oneshot", torch.bfloat16, dev)
                       for _ in range(R_)]
                g = capture(torch, lambda: [op(pp) for op, pp in zip(ops, ps)])
                for _ in range(3):
                    g.replay()
                reps = max(3, min(50, args.steps // 40))
                ms = time_graph_replays(torch, [g], reps) / (reps * R_)
                sim_more[f"tp{N_}"] = {"us": round(ms * 1e3, 3),
                                       "value": round(N_ * 2 * n / (ms * 1e-3) / 1e9, 1),
                                       "unit": UNIT,
                                       "hbm_gbs": round(per / (ms * 1e-3) / 1e9, 1)}
                del ps, ops, g
                torch.cuda.empty_cache()
        except Exception as exc:  # noqa: BLE001  (informational only)
            sim_more = {"error": f"{type(exc).__name__}: {exc}"[:200]}

    # ---- end to end through the public API with pinned host buffers:
    # HostPipeline (chunked H2D -> compressed all-reduce -> D2H on three
    # streams), the host-array-in / host-array-out shape of the reference API
    e2e = None
    if not args.no_e2e:
        from paper_2411_09510_b200.collective import HostPipeline

        host_in = [torch.from_numpy(host_parts[r]).to(torch.bfloat16).pin_memory() for r in mine]
        host_out = torch.empty(n, dtype=torch.bfloat16).pin_memory()
        w = [int(v) for v in args.e2e_pieces.split(",")]
        pieces = w[0] if len(w) == 1 else tuple(w)
        if sim:
            pipe = HostPipeline.simulated(sch, n, nranks, args.algo, torch.bfloat16, dev,
                                          chunks=pieces)
        else:
            # eager issue across ranks: no NCCL inside a multi-stream graph capture
            pipe = HostPipeline.compressed(sch, n, algo=args.algo, out_dtype=torch.bfloat16,
                                           device=dev, chunks=pieces, graph=False)
        ke = max(3, min(args.steps, 100))
        for _ in range(3):
            pipe(host_in, host_out)
        torch.cuda.synchronize()
        # the host result equals the device path's result bit for bit
        dparts = [h.to(dev) for h in host_in]
        ref = (SimulatedAllReduce(sch, n, nranks, args.algo, torch.bfloat16, dev)(dparts) if sim
               else CompressedAllReduce(sch, n, algo=args.algo, out_dtype=torch.bfloat16,
                                        device=dev)(dparts[0]))
        exact = bool(torch.equal(ref.reshape(-1).cpu().view(torch.int16), host_out.view(torch.int16)))
        del dparts, ref
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(ke):
            pipe(host_in, host_out)
        e1.record()
        torch.cuda.synchronize()
        ms_e = e0.elapsed_time(e1) / ke
        if world > 1:
            tt = torch.tensor([ms_e], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms_e = float(tt.item())
        e2e = {"value": round(nranks * 2 * n / (ms_e * 1e-3) / 1e9, 3), "unit": UNIT,
               "h2d_bytes_per_step": pipe.h2d_bytes, "d2h_bytes_per_step": pipe.d2h_bytes,
               "ms_per_step": round(ms_e, 4), "steps": ke, "pieces": pipe.k,
               "piece_values": [b1 - b0 for b0, b1 in zip(pipe.bounds, pipe.bounds[1:])],
               "bit_exact_vs_device_call": exact,
               "api": "HostPipeline.__call__ (pinned host partials -> pinned host result)"}

    # ---- uncompressed bf16 NCCL all-reduce on the same tensor (N>1)
    bf16_ar = None
    if world > 1:
        xs = [s_[0][0].clone() for s_ in sets]
        gsb = [capture(torch, (lambda x=x: dist.all_reduce(x))) for x in xs]
        for i in range(args.warmup):
            gsb[i % R].replay()
        dist.barrier()
        gsb_all = capture(torch, lambda: [dist.all_reduce(x) for x in xs])
        ms_b = time_steps(torch, gsb_all, gsb, args.steps) / args.steps
        tt = torch.tensor([ms_b], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_b = float(tt.item())
        bf16_ar = {"us": round(ms_b * 1e3, 2), "value": round(world * 2 * n / (ms_b * 1e-3) / 1e9, 2),
                   "unit": UNIT, "speedup_of_compressed": round(ms_b / ms_step, 3)}

    # ---- the NVLink-pull fused kernel over symmetric memory (N>1).  Every
    # stage that can fail agrees across ranks first (all_reduce MIN of an
    # ok flag), so one rank's failure can never leave the others waiting in
    # a collective.
    symm = None
    if world > 1 and os.environ.get("MXB200_BENCH_SYMM", "1") == "1":
        from paper_2411_09510_b200.collective import SymmetricAllReduce

        def all_ok(ok):
            t = torch.tensor([1 if ok else 0], device=dev, dtype=torch.int32)
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            return bool(t.item())

        err, sar, ms_s, exact = None, None, None, None
        try:
            sar = SymmetricAllReduce(sch, n, out_dtype=torch.bfloat16, device=dev, algo=args.algo)
            x0 = sets[0][0][0]
            got = sar(x0).clone()
            torch.cuda.synchronize()
            sar.check_status()
        except Exception as exc:  # noqa: BLE001
            err = exc
        ok = all_ok(err is None)  # identical on every rank
        if ok:
            one = CompressedAllReduce(sch, n, algo=args.algo, out_dtype=torch.bfloat16, device=dev)
            ref = one(x0).clone()
            exact = bool(torch.equal(got.view(torch.int16), ref.view(torch.int16)))
            try:
                gss = [capture(torch, (lambda x=s_[0][0]: sar(x))) for s_ in sets]
                for i in range(args.warmup):
                    gss[i % R].replay()
                torch.cuda.synchronize()
                gss_all = capture(torch, lambda: [sar(s_[0][0]) for s_ in sets])
                ms_s = time_steps(torch, gss_all, gss, args.steps) / args.steps
                sar.check_status()  # a timed-out peer wait invalidates the number
            except Exception as exc:  # noqa: BLE001
                err = exc
            ok = all_ok(err is None)
        if ok:
            tt = torch.tensor([ms_s], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms_s = float(tt.item())
            symm = {"us": round(ms_s * 1e3, 2),
                    "value": round(world * 2 * n / (ms_s * 1e-3) / 1e9, 2), "unit": UNIT,
                    f"bit_exact_vs_nccl_{args.algo}": exact,
                    "kernel": ("k_symm_flow (per-CTA: quantise -> release flag to every peer "
                               "-> acquire N flags -> NVLink pull dequant-sum; one launch per "
                               "rank, no grid barrier)" if args.algo == "oneshot" else
                               "k_symm2_flow (per-CTA: quantise N chunks -> flag -> pull my "
                               "chunk from N peers, fp32 sum, requantise -> flag -> pull N "
                               "reduced chunks, decode; one launch per rank)")}
            if bf16_ar:
                symm["speedup_vs_bf16_allreduce"] = round(bf16_ar["us"] / symm["us"], 3)
        else:
            symm = {"error": (f"{type(err).__name__}: {err}"[:300] if err is not None
                              else "failed on another rank")}

    # the collective against NVLink (N>1): effective (uncompressed-equivalent,
    # nccl-tests "algbw") and wire GB/s per rank, against 900 GB/s/direction
    coll = None
    if world > 1:
        wire = ((world - 1) * S if args.algo == "oneshot" else
                2 * (world - 1) * _native.shard_layout(
                    twoshot_chunk_values(n, world, sch.block_size), sch.to_c())[2])
        t = ms_step * 1e-3
        coll = {"effective_algbw_gbs": round(2 * n / t / 1e9, 1),
                "busbw_gbs": round(2 * n / t / 1e9 * 2 * (world - 1) / world, 1),
                "wire_bytes_per_rank": wire, "wire_gbs_per_rank": round(wire / t / 1e9, 1),
                "nvlink_gbs_per_direction": 900.0,
                "wire_frac_of_nvlink": round(wire / t / 1e9 / 900.0, 4)}

    if rank != 0:
        return
    cpu = None if (args.no_cpu_baseline or world > 1) else cpu_baseline(args.scheme, shape, nranks)
    line = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 5),
            "us_per_allreduce": round(ms_step * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (gaussian_with_outliers N(0,1) with 1% x100 outliers, "
                    "mx/synth.py), bf16 partial sums",
            "config": config_dict(args, shape, world),
            "wire_bytes_per_rank": ((nranks - 1) * S if args.algo == "oneshot" else
                                    2 * (nranks - 1) * _native.shard_layout(
                                        twoshot_chunk_values(n, nranks, sch.block_size),
                                        sch.to_c())[2]),
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps, "clocks": clocks,
            "bf16_nccl_allreduce": bf16_ar, "symmetric_memory_fused": symm,
            "collective": coll, "simulated_tp_fused_step": sim_more}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    shape = tuple(int(v) for v in args.shape.split(","))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.algo == "auto":
        tp = args.sim_ranks if world == 1 else world
        args.algo = "oneshot" if tp <= 2 else "twoshot"
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, shape, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, shape, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
