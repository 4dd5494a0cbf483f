"""Cost of the all-gather riding on the GEMM epilogue (one B200): the fused
GEMM + quantiser writing its shard once (local) against the push GEMM
writing it into npush rank buffers (here all on this device, so the bytes go
to HBM instead of NVLink -- an upper bound on the epilogue's extra store
work) plus its end-of-kernel publish.  CUDA-graph replays, operand sets
rotated beyond L2; us per GEMM.

    python scripts/push_bench.py [scheme ...]   (default fp4_e2m1:32:e8m0)
"""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2411_09510_b200 import _native  # noqa: E402
from paper_2411_09510_b200.formats import parse_scheme  # noqa: E402
from scripts.gemm_bench import time_graph  # noqa: E402

L2 = 126 * 1024 * 1024


def main():
    lib = _native.load()
    for spec in sys.argv[1:] or ["fp4_e2m1:32:e8m0"]:
        run(lib, spec)


def run(lib, spec):
    cs = parse_scheme(spec).to_c()
    P = ctypes.c_void_p
    st = lambda: P(torch.cuda.current_stream().cuda_stream)  # noqa: E731
    for label, M, N, K in (("8b o_proj tp2", 2048, 4096, 2048), ("8b down_proj tp2", 2048, 4096, 7168),
                           ("8b o_proj tp8", 2048, 4096, 512), ("70b o_proj tp8", 4096, 8192, 1024)):
        per = 2 * (M * K + N * K)
        R = max(2, -(-3 * L2 // per))
        xs = [torch.randn(M, K, device="cuda").to(torch.bfloat16) for _ in range(R)]
        ws = [(torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16) for _ in range(R)]
        so, eo, S = _native.shard_layout(M * N, cs)
        shard = torch.empty(S, dtype=torch.uint8, device="cuda")
        res = {"scheme": spec, "shape": label, "M": M, "N": N, "K": K}

        def local(i):
            _native.check(lib.mx_gemm_quantize(P(xs[i].data_ptr()), P(ws[i].data_ptr()), M, N, K,
                                               ctypes.byref(cs), P(shard.data_ptr() + so),
                                               P(shard.data_ptr() + eo), None, None, st()), "g")
        res["fused_local_us"] = round(time_graph(local, R), 2)
        out = torch.empty(M * N, dtype=torch.bfloat16, device="cuda")

        def local_pair(i):  # fused GEMM + K2 over the one shard (world 1, no exchange)
            local(i)
            _native.check(lib.mx_dequant_sum(P(shard.data_ptr()), S, 1, M * N, M * N, 0,
                                             ctypes.byref(cs), P(out.data_ptr()), _native.MX_BF16,
                                             st()), "k2")
        res["fused_local_plus_k2_us"] = round(time_graph(local_pair, R), 2)
        for npush in (1, 2, 4, 8):
            slot, sh, foff, total = _native.push_layout(M * N, cs, npush)
            bufs = [torch.zeros(total, dtype=torch.uint8, device="cuda") for _ in range(npush)]
            bptr = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device="cuda")
            fptr = torch.tensor([b.data_ptr() + foff for b in bufs], dtype=torch.int64,
                                device="cuda")
            state = torch.zeros(4, dtype=torch.int32, device="cuda")

            def push(i):
                _native.check(lib.mx_gemm_allgather_push(
                    P(xs[i].data_ptr()), P(ws[i].data_ptr()), M, N, K, ctypes.byref(cs),
                    P(bptr.data_ptr()), 0, npush, P(state.data_ptr() + 4), None, st()), "push")
            res[f"push{npush}_us"] = round(time_graph(push, R), 2)
            if npush == 1:
                def pair(i):  # push GEMM (+ publish) -> wait / decode (world 1)
                    push(i)
                    _native.check(lib.mx_push_dequant_sum(
                        P(bufs[0].data_ptr()), M * N, ctypes.byref(cs), 0, 1,
                        P(bufs[0].data_ptr() + foff), P(state.data_ptr() + 4), P(state.data_ptr()),
                        P(out.data_ptr()), _native.MX_BF16, None, st()), "decode")
                res["push1_plus_decode_us"] = round(time_graph(pair, R), 2)
            del bufs
        print(json.dumps(res), flush=True)
        del xs, ws
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
