"""BASELINE.json configs[3] and configs[4] on one B200.

  python scripts/sweeps.py formats   # MXFP4/5/6/INT8 x block 16/32/64, E8M0, [2048x4096]
  python scripts/sweeps.py messages  # 64 KiB .. 512 MiB bf16 messages

formats: per scheme -- K1 and K2 (2 shards) device time and HBM GB/s, the
fused simulated-TP=2 step, the wire payload, and the error of the reduced
tensor (MX one-shot, fp32 rank-order sum, bf16 cast) against the exact
fp64 sum of the two bf16 partials: SQNR, max-abs, MSE.  The GPU result is
bit-identical to the reference's own dequantised sum (tests/), so these are
also the reference's errors.

messages: per size -- K1, K2 and the fused step (simulated TP=2), plus the
analytic NVLink wire time at TP=2/4/8 for one-shot / two-shot / bf16 ring,
using 770 GB/s per direction (the measured peer-copy reference of
B200_PROFILING.md).  Multi-GPU collectives are not measurable with one GPU;
the model lines are labelled as such.

One JSON line per configuration on stdout.
"""

import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2411_09510_b200 import _native  # noqa: E402
from paper_2411_09510_b200.collective import NativeBackend, SimulatedAllReduce  # noqa: E402
from paper_2411_09510_b200.formats import parse_scheme  # noqa: E402
from paper_2411_09510_b200.synth import rank_partials  # noqa: E402

L2 = 126 * 2 ** 20
NVLINK_GBS = 770.0


def graph_time(fn, reps):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(g):
        fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def kernel_times(spec, parts, R):
    """(us K1, us K2-2shards, us fused step) over R rotated buffer sets."""
    sch = parse_scheme(spec, extensions=True)
    n = parts[0][0].numel()
    be = NativeBackend(sch)
    sets = [SimulatedAllReduce(sch, n, 2, "oneshot", torch.bfloat16) for _ in range(R)]
    for op, p in zip(sets, parts):
        op(p)  # fill shards
    reps = max(3, min(50, int(2e4 / max(1, R))))
    k1 = graph_time(lambda: [be.quantize_into(p[0].reshape(-1), op.gathered[:op.S], op.ws, op.flag)
                             for op, p in zip(sets, parts)], reps) / R
    k2 = graph_time(lambda: [op.reduce() for op in sets], reps) / R
    step = graph_time(lambda: [op(p) for op, p in zip(sets, parts)], reps) / R
    return k1 * 1e3, k2 * 1e3, step * 1e3, sets[0].S, sets[0].fused


def formats(grid=None):
    T, H = 2048, 4096
    n = T * H
    host = rank_partials((T, H), 2, seed=0)
    exact = host[0].astype(np.float64) + host[1].astype(np.float64)
    base = [torch.from_numpy(h).to("cuda", torch.bfloat16) for h in host]
    R = max(2, -(-3 * L2 // (6 * n)))
    parts = [[(b.roll(i * 7, 0) * (-1) ** i).contiguous() for b in base] for i in range(R)]
    if grid is None:  # BASELINE configs[3]
        grid = [f"{el}:{B}:e8m0" for el in ["fp4_e2m1", "fp5_e2m2", "fp6_e2m3", "int8"]
                for B in (16, 32, 64)]
    for spec in grid:
        if True:
            k1, k2, step, S, fused = kernel_times(spec, parts, R)
            op = SimulatedAllReduce(spec, n, 2, "oneshot", torch.float32)
            red = op(base).double().cpu().numpy().reshape(T, H)
            err = red - exact
            sch = parse_scheme(spec, extensions=True)
            sb, eb = _native.stream_nbytes(n, sch.to_c())
            print(json.dumps({
                "config": "formats", "scheme": spec, "shape": [T, H],
                "k1_us": round(k1, 3), "k1_gbs": round((2 * n + sb + eb) / k1 / 1e3, 1),
                "k2_us": round(k2, 3), "k2_gbs": round((2 * (sb + eb) + 2 * n) / k2 / 1e3, 1),
                "fused_step_us": round(step, 3), "fused": fused,
                "payload_bytes": sb + eb, "ratio_vs_bf16": round(2 * n / (sb + eb), 3),
                "sqnr_db": round(10 * math.log10(float((exact ** 2).sum() / (err ** 2).sum())), 3),
                "max_abs_err": float(np.abs(err).max()), "mse": float((err ** 2).mean())}),
                flush=True)


def paper():
    """The paper's own grid (mx/search.py TABLE1: fp3_e1m1 / fp4_e2m1 /
    fp5_e2m2 x block 8/16/32, E5M0 scales) plus the same formats with E8M0."""
    formats([f"{el}:{B}:{sc}" for sc in ("e5m0", "e8m0") for el in ("fp3_e1m1", "fp4_e2m1", "fp5_e2m2")
             for B in (8, 16, 32)])


def wire_model(n, S, N):
    """Per-GPU per-direction bytes and modelled time at NVLINK_GBS."""
    one = (N - 1) * S
    two = 2 * (N - 1) * S / N
    ring = 2 * (N - 1) / N * 2 * n
    us = lambda b: b / NVLINK_GBS / 1e3  # noqa: E731
    return {"oneshot_bytes": one, "twoshot_bytes": int(two), "bf16_ring_bytes": int(ring),
            "oneshot_wire_us": round(us(one), 2), "twoshot_wire_us": round(us(two), 2),
            "bf16_ring_wire_us": round(us(ring), 2)}


def messages():
    spec = "fp4_e2m1:32:e8m0"
    for lg in range(15, 29):
        n = 1 << lg
        R = max(1, min(64, -(-3 * L2 // (6 * n))))
        g = torch.Generator(device="cuda").manual_seed(lg)
        base = [torch.randn(n, device="cuda", generator=g).to(torch.bfloat16) for _ in range(2)]
        parts = [[(b.roll(i * 17) * (-1) ** i).contiguous() for b in base] for i in range(R)]
        k1, k2, step, S, fused = kernel_times(spec, parts, R)
        line = {"config": "messages", "scheme": spec, "bf16_bytes": 2 * n, "rotation": R,
                "k1_us": round(k1, 3), "k2_us": round(k2, 3), "fused_step_us": round(step, 3),
                "fused": fused, "shard_bytes": S,
                "model_nvlink": {f"tp{N}": wire_model(n, S, N) for N in (2, 4, 8)},
                "model_note": f"wire time = bytes / {NVLINK_GBS} GB/s per direction (model)"}
        print(json.dumps(line), flush=True)
        del parts, base
        torch.cuda.empty_cache()


def tp():
    """Per-rank device cost of the compressed collective at TP = 2/4/8,
    measured on one GPU with the real kernels (a rank's K1, and K2 over N
    shards / the two-shot K1-chunked + K3 + K2 chain), next to the NVLink
    wire time of its bytes at NVLINK_GBS (model; one GPU cannot measure the
    exchange).  8B and 70B prefill shapes, fp4_e2m1:32:e8m0."""
    from paper_2411_09510_b200.collective import chunk_len, twoshot_chunk_values

    spec = "fp4_e2m1:32:e8m0"
    sch = parse_scheme(spec, extensions=True)
    be = NativeBackend(sch)
    for T, H in ((2048, 4096), (4096, 8192)):
        n = T * H
        for N in (2, 4, 8):
            R = max(2, -(-3 * L2 // ((N + 2) * n)))
            g = torch.Generator(device="cuda").manual_seed(N)
            xs = [torch.randn(n, device="cuda", generator=g).to(torch.bfloat16) for _ in range(R)]
            ops1 = [SimulatedAllReduce(sch, n, N, "oneshot", torch.bfloat16, fused=False)
                    for _ in range(R)]
            for op, x in zip(ops1, xs):
                op([x] * N)
            reps = max(3, min(50, int(2e3 / R)))
            k1 = graph_time(lambda: [be.quantize_into(x, op.gathered[:op.S], op.ws, op.flag)
                                     for op, x in zip(ops1, xs)], reps) / R
            k2 = graph_time(lambda: [op.reduce() for op in ops1], reps) / R
            S = ops1[0].S
            del ops1
            ops2 = [SimulatedAllReduce(sch, n, N, "twoshot", torch.bfloat16) for _ in range(R)]
            for op, x in zip(ops2, xs):
                op([x] * N)
            c, S2 = ops2[0].c, ops2[0].S
            own = chunk_len(n, c, 0)
            t_q = graph_time(lambda: [be.quantize_chunks(x, c, op.send[0], S2, op.ws, op.flag)
                                      for op, x in zip(ops2, xs)], reps) / R
            t_r = graph_time(lambda: [be.requant(op.recv[0], S2, N, own, c, op.gathered[:S2],
                                                 op.ws, op.flag) for op in ops2], reps) / R
            t_d = graph_time(lambda: [be.dequant_sum(op.gathered, 0, 1, n, c, S2, op.out)
                                      for op in ops2], reps) / R
            del ops2, xs
            torch.cuda.empty_cache()
            wm = wire_model(n, S, N)
            one = (k1 + k2) * 1e3
            two = (t_q + t_r + t_d) * 1e3
            print(json.dumps({
                "config": "tp", "scheme": spec, "shape": [T, H], "tp": N,
                "oneshot_us": {"k1": round(k1 * 1e3, 3), "k2_nshards": round(k2 * 1e3, 3),
                               "compute": round(one, 3), "wire_model": wm["oneshot_wire_us"],
                               "total_model": round(one + wm["oneshot_wire_us"], 2)},
                "twoshot_us": {"k1_chunked": round(t_q * 1e3, 3), "k3_requant": round(t_r * 1e3, 3),
                               "k2_final": round(t_d * 1e3, 3), "compute": round(two, 3),
                               "wire_model": wm["twoshot_wire_us"],
                               "total_model": round(two + wm["twoshot_wire_us"], 2)},
                "bf16_ring_wire_model_us": wm["bf16_ring_wire_us"],
                "note": f"kernel times measured on one B200; wire = bytes / {NVLINK_GBS} GB/s "
                        "(model, no overlap assumed)"}), flush=True)


def codecs():
    """Paper Table 4 on one B200: MX vs the comparison codecs (channel-wise
    INT, TopK) vs fp16 on the 8B prefill partial, simulated TP=2.  Device
    compress / decompress time of one rank's partial, wire payload, and the
    error of the float64 rank-order sum of the decoded partials against the
    exact sum (the tpsim report, mx/tpsim.py:234-302)."""
    from paper_2411_09510_b200 import baselines as bl
    from paper_2411_09510_b200.codec import (compress_tensor_device, decompress_tensor_device,
                                             header_nbytes)

    T, H = 2048, 4096
    n = T * H
    host = rank_partials((T, H), 2, seed=0)
    exact = host[0].astype(np.float64) + host[1].astype(np.float64)
    base = [torch.from_numpy(h).to("cuda", torch.bfloat16) for h in host]
    R = max(2, -(-3 * L2 // (3 * n)))
    xs = [(base[0].roll(i * 7, 0) * (-1) ** i).contiguous() for i in range(R)]

    def mx_codec(spec):
        sch = parse_scheme(spec, extensions=True)
        enc = lambda x: compress_tensor_device(x, sch, check_finite=False)  # noqa: E731
        dec = lambda c: decompress_tensor_device(c, torch.bfloat16)  # noqa: E731
        sb, eb = _native.stream_nbytes(n, sch.to_c())
        return enc, dec, header_nbytes(2) + sb + eb

    def chan(bits):
        enc = lambda x: bl.channelwise_int_compress_device(x, bits, check_finite=False)  # noqa: E731
        dec = lambda c: bl.channelwise_int_decompress_device(c[0], c[1], c[2], bits,  # noqa: E731
                                                             torch.bfloat16)
        return enc, dec, header_nbytes(2) + 2 * H + (n * bits + 7) // 8

    def topk(f):
        k = bl.topk_budget(n, 2, f)
        enc = lambda x: bl.topk_compress_device(x, k, check_finite=False)  # noqa: E731
        dec = lambda c: bl.topk_decompress_device(c[0], c[1], n, torch.bfloat16)  # noqa: E731
        return enc, dec, header_nbytes(2) + 6 * k

    def fp16():
        return (lambda x: x.to(torch.float16)), (lambda c: c.to(torch.bfloat16)), \
            header_nbytes(2) + 2 * n

    table = [("fp4_e2m1:32:e8m0", mx_codec("fp4_e2m1:32:e8m0")),
             ("fp6_e2m3:32:e8m0", mx_codec("fp6_e2m3:32:e8m0")),
             ("chanint:4", chan(4)), ("chanint:8", chan(8)),
             ("topk:3", topk(3.0)), ("topk:10", topk(10.0)), ("fp16", fp16())]
    for name, (enc, dec, payload) in table:
        comp = [enc(x) for x in xs]
        reps = 20
        t_enc = graph_time(lambda: [enc(x) for x in xs], reps) / R
        t_dec = graph_time(lambda: [dec(c) for c in comp], reps) / R
        rec = [dec(enc(b)).double().cpu().numpy().reshape(T, H) for b in base]
        err = rec[0] + rec[1] - exact
        print(json.dumps({
            "config": "codecs", "codec": name, "shape": [T, H], "tp": 2,
            "compress_us": round(t_enc * 1e3, 3), "decompress_us": round(t_dec * 1e3, 3),
            "payload_bytes": payload, "ratio_vs_bf16": round(2 * n / payload, 3),
            "rel_frob_err": float(np.linalg.norm(err) / np.linalg.norm(exact)),
            "sqnr_db": round(10 * math.log10(float((exact ** 2).sum() / (err ** 2).sum())), 3),
            "max_abs_err": float(np.abs(err).max()),
            "note": "decoded to bf16 for timing; errors from the float64 rank-order sum "
                    "of the decoded partials (bf16 output rounding included)"}), flush=True)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "formats"
    {"formats": formats, "messages": messages, "codecs": codecs, "tp": tp, "paper": paper}[what]()
