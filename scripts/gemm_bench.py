"""Row-parallel GEMM + MX quantise at the Llama prefill shapes (one B200).

For each (model, projection, TP) shape x[M, K] . W[N, K]^T it times, with
CUDA events over CUDA-graph replays of buffer sets rotated beyond L2 (so W
streams from HBM as in a real layer stack):
  cublas        torch F.linear (cuBLAS bf16 GEMM), bf16 partial out
  cublas+k1     F.linear then K1 (mx_quantize) into the shard: the unfused
                producer of the compressed all-reduce
  ours_plain    k_gemm_mx plain mode (bf16 partial out)
  ours_fused    k_gemm_mx with the quantiser in the epilogue (shard only)
and reports us, TFLOP/s and the fraction of the measured bf16 peak.

    python scripts/gemm_bench.py [--shapes 8b,70b] [--spec fp4_e2m1:32:e8m0]
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

L2 = 126 * 1024 * 1024

SHAPES = {
    # (label, M tokens, N hidden, K local in-features)
    "8b": [("llama-3.1-8b o_proj tp2", 2048, 4096, 2048),
           ("llama-3.1-8b down_proj tp2", 2048, 4096, 7168),
           ("llama-3.1-8b o_proj tp8", 2048, 4096, 512),
           ("llama-3.1-8b down_proj tp8", 2048, 4096, 1792)],
    "8b_tp1": [("llama-3.1-8b o_proj tp1", 2048, 4096, 4096),
               ("llama-3.1-8b down_proj tp1", 2048, 4096, 14336)],
    "70b": [("llama-3.1-70b o_proj tp8", 4096, 8192, 1024),
            ("llama-3.1-70b down_proj tp8", 4096, 8192, 3584)],
}


def peak_tflops():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"], "measured"
    except Exception:  # noqa: BLE001
        return 1590.0, "fallback"


def time_graph(fn, R, reps=20):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(R):
            fn(i)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for i in range(R):
            fn(i)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(100_000)
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / (reps * R))
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="8b,70b")
    ap.add_argument("--spec", default="fp4_e2m1:32:e8m0")
    ap.add_argument("--filter", default="", help="only shapes whose label contains this")
    ap.add_argument("--variants", default="cublas,cublas+k1,ours_plain,ours_fused")
    ap.add_argument("--profile", action="store_true", help="ncu mode: one launch of each variant")
    args = ap.parse_args()
    from paper_2411_09510_b200 import _native
    from paper_2411_09510_b200.formats import parse_scheme

    lib = _native.load()
    cs = parse_scheme(args.spec, extensions=True).to_c()
    peak, kind = peak_tflops()
    st = lambda: ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    for tag in args.shapes.split(","):
        for label, M, N, K in SHAPES[tag]:
            if args.filter not in label:
                continue
            per = 2 * (M * K + N * K + M * N)
            R = max(2, -(-3 * L2 // per))
            xs = [torch.randn(M, K, device="cuda").to(torch.bfloat16) for _ in range(R)]
            ws = [(torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
                  for _ in range(R)]
            outs = [torch.empty(M, N, device="cuda", dtype=torch.bfloat16) for _ in range(R)]
            sb, eb = _native.stream_nbytes(M * N, cs)
            so, eo, S = _native.shard_layout(M * N, cs)
            shards = [torch.empty(S, device="cuda", dtype=torch.uint8) for _ in range(R)]
            wsz = _native.workspace_bytes(M * N, cs, False)
            wsb = torch.empty(max(wsz, 1), device="cuda", dtype=torch.uint8)

            def cublas(i):
                torch.matmul(xs[i], ws[i].T, out=outs[i])

            def cublas_k1(i):
                torch.matmul(xs[i], ws[i].T, out=outs[i])
                _native.check(lib.mx_quantize(
                    P(outs[i]), _native.MX_BF16, M * N, ctypes.byref(cs),
                    ctypes.c_void_p(shards[i].data_ptr() + so),
                    ctypes.c_void_p(shards[i].data_ptr() + eo), None, P(wsb), wsb.numel(), st()),
                    "mx_quantize")

            def plain(i, sk=True):
                _native.check(lib.mx_gemm_quantize(
                    P(xs[i]), P(ws[i]), M, N, K, None, None, None, P(outs[i]), None,
                    st()), "gemm")

            def fused(i, sk=True):
                _native.check(lib.mx_gemm_quantize(
                    P(xs[i]), P(ws[i]), M, N, K, ctypes.byref(cs),
                    ctypes.c_void_p(shards[i].data_ptr() + so),
                    ctypes.c_void_p(shards[i].data_ptr() + eo), None, None,
                    st()), "gemm")

            flops = 2.0 * M * N * K
            row = {"shape": label, "M": M, "N": N, "K": K, "spec": args.spec, "rotation": R,
                   "peak_tflops": peak, "peak_kind": kind}
            variants = (("cublas", cublas), ("cublas+k1", cublas_k1), ("ours_plain", plain),
                        ("ours_fused", fused))
            if args.profile:
                for name, fn in variants:
                    if name in args.variants.split(","):
                        fn(0)
                        fn(1)
                torch.cuda.synchronize()
                continue
            for name, fn in variants:
                if name not in args.variants.split(","):
                    continue
                try:
                    us = time_graph(fn, R)
                    tf = flops / (us * 1e-6) / 1e12
                    row[name] = {"us": round(us, 2), "tflops": round(tf, 1),
                                 "frac": round(tf / peak, 3)}
                except Exception as exc:  # noqa: BLE001
                    row[name] = {"error": f"{type(exc).__name__}: {exc}"[:200]}
            # parity of this shape: fused shard == K1 of our own plain partial
            try:
                plain(0)
                ref = torch.empty_like(shards[0])
                _native.check(lib.mx_quantize(
                    P(outs[0]), _native.MX_BF16, M * N, ctypes.byref(cs),
                    ctypes.c_void_p(ref.data_ptr() + so), ctypes.c_void_p(ref.data_ptr() + eo),
                    None, P(wsb), wsb.numel(), st()), "mx_quantize")
                fused(0)
                torch.cuda.synchronize()
                row["fused_shard_equals_k1_of_partial"] = bool(
                    torch.equal(ref[so:so + sb], shards[0][so:so + sb])
                    and torch.equal(ref[eo:eo + eb], shards[0][eo:eo + eb]))
                ref32 = xs[0].float() @ ws[0].float().T
                row["plain_max_rel_err_vs_fp32"] = float(
                    ((outs[0].float() - ref32).abs().max() / ref32.abs().max()).item())
            except Exception as exc:  # noqa: BLE001
                row["parity_error"] = f"{type(exc).__name__}: {exc}"[:200]
            if "us" in row.get("ours_fused", {}) and "us" in row.get("cublas+k1", {}):
                row["fused_speedup_vs_cublas_k1"] = round(
                    row["cublas+k1"]["us"] / row["ours_fused"]["us"], 3)
            print(json.dumps(row), flush=True)
            del xs, ws, outs, shards
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
