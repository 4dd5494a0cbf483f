"""Where the push decode's extra time goes at world size 1 (one B200):
K2 over one shard, against mx_push_dequant_sum on the same shard with its
flag already set (an immediately satisfied wait + decode),
and against the full push GEMM + decode pair.  CUDA-graph replays.

    python scripts/push_handshake.py
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


def main():
    lib = _native.load()
    P = ctypes.c_void_p
    st = lambda: P(torch.cuda.current_stream().cuda_stream)  # noqa: E731
    for spec in sys.argv[1:] or ["fp4_e2m1:32:e8m0"]:
        cs = parse_scheme(spec).to_c()
        for M, N, K in ((2048, 4096, 2048), (4096, 8192, 1024)):
            n = M * N
            x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
            w = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
            slot, sh, foff, total = _native.push_layout(n, cs, 1)
            buf = torch.zeros(total, dtype=torch.uint8, device="cuda")
            bptr = torch.tensor([buf.data_ptr()], dtype=torch.int64, device="cuda")
            fptr = torch.tensor([buf.data_ptr() + foff], dtype=torch.int64, device="cuda")
            state = torch.zeros(4, dtype=torch.int32, device="cuda")
            out = torch.empty(n, dtype=torch.bfloat16, device="cuda")

            def gemm(i):
                _native.check(lib.mx_gemm_allgather_push(
                    P(x.data_ptr()), P(w.data_ptr()), M, N, K, ctypes.byref(cs), P(bptr.data_ptr()),
                    0, 1, P(state.data_ptr() + 4), None, st()), "push")

            def decode(i):
                _native.check(lib.mx_push_dequant_sum(
                    P(buf.data_ptr()), n, ctypes.byref(cs), 0, 1,
                    P(buf.data_ptr() + foff), P(state.data_ptr() + 4), P(state.data_ptr()),
                    P(out.data_ptr()), _native.MX_BF16, None, st()), "decode")

            def k2(i):  # the same shard (slot 1 after one push), plain K2
                _native.check(lib.mx_dequant_sum(P(base), sh, 1, n, n, 0, ctypes.byref(cs),
                                                 P(out.data_ptr()), _native.MX_BF16, st()), "k2")

            gemm(0)
            decode(0)
            torch.cuda.synchronize()
            base = buf.data_ptr() + (int(state[1].item()) & 1) * slot
            res = {"scheme": spec, "M": M, "N": N, "K": K,
                   "k2_us": round(time_graph(k2, 8), 2),
                   "decode_flag_set_us": round(time_graph(decode, 8), 2),
                   "push_gemm_us": round(time_graph(gemm, 4), 2),
                   "push_gemm_plus_decode_us": round(time_graph(lambda i: (gemm(i), decode(i)), 4), 2)}
            assert int(state[0].item()) == 0
            print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
