"""GPU: the peer-memory collectives across separate PROCESSES on one device.

Every other multi-rank GPU test runs its ranks as concurrent launches of
ONE process.  Here each rank is its own process with its own CUDA context
and streams, as on a real TP node: rank r allocates its collective buffer,
the buffers are exchanged as CUDA IPC mappings (torch.multiprocessing
shares CUDA tensors through cudaIpcGetMemHandle / cudaIpcOpenMemHandle,
the mechanism symmetric memory uses across GPUs), and the kernels run
through the C ABI with those peer pointers: the NVLink one-shot / two-shot
(K5 / K5b) and the GEMM push (one-shot and two-shot).  Stores from one
context, flags released at system scope, acquired in the other: every
rank's result equals the oracle's all-reduce of the two ranks' partials,
over repeated calls (both slots, twice), at 2 and 4 processes.  (torch's
own symmetric memory refuses two ranks on one device, hence the IPC
exchange; kernels of different contexts time-slice on the GPU, so every
flag wait also survives preemption.)"""

import ctypes
import os
import socket
import traceback

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CALLS = 4


def _worker(rank, WORLD, port, qs):
    try:
        os.environ["MXB200_SYMM_TIMEOUT_MS"] = "20000"
        import torch.distributed as dist

        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=WORLD)
        from oracle import mx_oracle as O
        from paper_2411_09510_b200 import _native
        from paper_2411_09510_b200.formats import parse_scheme

        lib = _native.load()
        P = ctypes.c_void_p
        res = {}

        def exchange(buf, tag):
            """rank-ordered list of every rank's buffer (peer ones IPC-mapped)"""
            for r in range(WORLD):
                if r != rank:
                    qs[(rank, r)].put((tag, buf))
            got = {rank: buf}
            for r in range(WORLD):
                if r != rank:
                    t, b = qs[(r, rank)].get(timeout=120)
                    assert t == tag
                    got[r] = b
            return [got[r] for r in range(WORLD)]

        def gather(t):
            allt = [torch.empty_like(t) for _ in range(WORLD)]
            dist.all_gather(allt, t)
            return allt

        st = torch.cuda.Stream()
        # ---- K5 / K5b: the NVLink one-shot / two-shot kernels
        n = 64 * 1024
        for spec in ("fp4_e2m1:32:e8m0", "fp5_e2m2:32:e5m0"):
            cs = parse_scheme(spec).to_c()
            for algo in ("oneshot", "twoshot"):
                if algo == "oneshot":
                    slot, foff, total, ctas = _native.symm_layout(n, cs, WORLD)
                else:
                    slot, _, foff, total, ctas = _native.symm_twoshot_layout(n, cs, WORLD)
                buf = torch.zeros(total, dtype=torch.uint8, device="cuda")
                torch.cuda.synchronize()
                bufs = exchange(buf, f"symm-{spec}-{algo}")
                bptr = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device="cuda")
                fptr = torch.tensor([b.data_ptr() + foff for b in bufs], dtype=torch.int64,
                                    device="cuda")
                state = torch.zeros(1 + ctas, dtype=torch.int32, device="cuda")
                nf = torch.empty(1, dtype=torch.int64, device="cuda")
                lib.mx_nonfinite_reset(P(nf.data_ptr()), None)
                out = torch.empty(n, dtype=torch.float32, device="cuda")
                dist.barrier()
                ok = True
                for c in range(CALLS):
                    g = torch.Generator().manual_seed(1000 * c + rank)
                    x = torch.randn(n, generator=g).to(torch.bfloat16)
                    host = [t.float().numpy().astype(np.float64) for t in gather(x)]
                    f = O.allreduce_oneshot if algo == "oneshot" else O.allreduce_twoshot
                    want = np.asarray(f(host, O.scheme(spec)), np.float32)
                    xd = x.cuda()
                    torch.cuda.synchronize()
                    common = (P(state.data_ptr()), P(state.data_ptr() + 4), P(nf.data_ptr()),
                              P(st.cuda_stream))
                    if algo == "oneshot":
                        rc = lib.mx_allreduce_symm(P(xd.data_ptr()), _native.MX_BF16, n,
                                                   ctypes.byref(cs), P(bptr.data_ptr()),
                                                   P(fptr.data_ptr()), rank, WORLD, slot,
                                                   P(out.data_ptr()), _native.MX_F32, None,
                                                   *common)
                    else:
                        rc = lib.mx_allreduce_symm_twoshot(P(xd.data_ptr()), _native.MX_BF16, n,
                                                           ctypes.byref(cs), P(bptr.data_ptr()),
                                                           P(fptr.data_ptr()), rank, WORLD,
                                                           P(out.data_ptr()), _native.MX_F32,
                                                           None, *common)
                    _native.check(rc, "symm")
                    st.synchronize()
                    ok &= int(state[0].item()) == 0
                    ok &= bool(np.array_equal(out.cpu().numpy(), want))
                res[f"symm {spec} {algo}"] = ok
                dist.barrier()
                del bufs
        # ---- the GEMM push, one-shot and two-shot
        M, N, K = 256, 512, 256
        nn = M * N
        for spec in ("fp4_e2m1:32:e8m0", "fp4_e2m1:8:e5m0", "fp5_e2m2:32:e5m0"):
            cs = parse_scheme(spec).to_c()
            for algo in ("oneshot", "twoshot"):
                if algo == "oneshot":
                    slot, sh, foff, total = _native.push_layout(nn, cs, WORLD)
                else:
                    _c, slot, sh, foff, total = _native.push2_layout(nn, cs, WORLD)
                buf = torch.zeros(total, dtype=torch.uint8, device="cuda")
                torch.cuda.synchronize()
                bufs = exchange(buf, f"push-{spec}-{algo}")
                bptr = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device="cuda")
                fptr = torch.tensor([b.data_ptr() + foff for b in bufs], dtype=torch.int64,
                                    device="cuda")
                state = torch.zeros(4, dtype=torch.int32, device="cuda")
                nf = torch.full((1,), -1, dtype=torch.int64, device="cuda")
                out = torch.empty(nn, dtype=torch.bfloat16, device="cuda")
                part = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
                dist.barrier()
                ok = True
                for c in range(CALLS):
                    g = torch.Generator().manual_seed(7000 + 100 * c + rank)
                    x = torch.randn(M, K, generator=g).to(torch.bfloat16).cuda()
                    w = (torch.randn(N, K, generator=g) / 16).to(torch.bfloat16).cuda()
                    _native.check(lib.mx_gemm_quantize(P(x.data_ptr()), P(w.data_ptr()), M, N, K,
                                                       None, None, None, P(part.data_ptr()), None,
                                                       P(st.cuda_stream)), "partial")
                    st.synchronize()
                    host = [t.float().numpy().ravel().astype(np.float64)
                            for t in gather(part.cpu())]
                    f = O.allreduce_oneshot if algo == "oneshot" else O.allreduce_twoshot
                    want = torch.from_numpy(np.asarray(f(host, O.scheme(spec)), np.float32)).to(
                        torch.bfloat16)
                    base = state.data_ptr()
                    if algo == "oneshot":
                        _native.check(lib.mx_gemm_allgather_push(
                            P(x.data_ptr()), P(w.data_ptr()), M, N, K, ctypes.byref(cs),
                            P(bptr.data_ptr()), rank, WORLD, P(base + 4), P(nf.data_ptr()),
                            P(st.cuda_stream)), "push")
                        _native.check(lib.mx_push_dequant_sum(
                            P(buf.data_ptr()), nn, ctypes.byref(cs), rank, WORLD,
                            P(buf.data_ptr() + foff), P(base + 4), P(base), P(out.data_ptr()),
                            _native.MX_BF16, None, P(st.cuda_stream)), "decode")
                    else:
                        _native.check(lib.mx_gemm_reducescatter_push(
                            P(x.data_ptr()), P(w.data_ptr()), M, N, K, ctypes.byref(cs),
                            P(bptr.data_ptr()), rank, WORLD, P(base + 4), P(nf.data_ptr()),
                            P(st.cuda_stream)), "push2")
                        _native.check(lib.mx_push2_requant(
                            P(buf.data_ptr()), nn, ctypes.byref(cs), rank, WORLD,
                            P(bptr.data_ptr()), P(fptr.data_ptr()), P(base + 4), P(base),
                            P(nf.data_ptr()), P(st.cuda_stream)), "requant")
                        _native.check(lib.mx_push2_decode(
                            P(buf.data_ptr()), nn, ctypes.byref(cs), rank, WORLD, P(base + 4),
                            P(base), P(out.data_ptr()), _native.MX_BF16, None,
                            P(st.cuda_stream)), "decode2")
                    st.synchronize()
                    ok &= int(state[0].item()) == 0
                    ok &= bool(torch.equal(out.cpu(), want))
                res[f"push {spec} {algo}"] = ok
                dist.barrier()
                del bufs
        dist.barrier()
        dist.destroy_process_group()
        outq = qs["out"]
        outq.put((rank, res))
    except Exception:  # noqa: BLE001
        qs["out"].put((rank, traceback.format_exc()[-4000:]))


@pytest.mark.parametrize("WORLD", [2, 4])
def test_processes_peer_collectives(WORLD):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    qs = {(a, b): ctx.Queue() for a in range(WORLD) for b in range(WORLD) if a != b}
    qs["out"] = ctx.Queue()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ps = [ctx.Process(target=_worker, args=(r, WORLD, port, qs)) for r in range(WORLD)]
    for p in ps:
        p.start()
    try:
        got = dict(qs["out"].get(timeout=300) for _ in ps)
    finally:
        for p in ps:
            p.join(timeout=120)
            if p.is_alive():
                p.kill()
    for r in range(WORLD):
        assert isinstance(got[r], dict), got[r]
        bad = [k for k, v in got[r].items() if not v]
        assert not bad, (r, bad)
        assert len(got[r]) == 10, got[r]
