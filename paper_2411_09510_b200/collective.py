"""Compressed tensor-parallel all-reduce over NCCL (NVLink 5 / NVSwitch).

Replaces the reference's threaded full-mesh exchange ``netbench._worker_loop``
(mx/netbench.py:307-339): every rank quantises its partial sum (its own
contribution included, mx/netbench.py:323), the packed shards cross the TP
group, and every rank decodes and sums all N contributions in fp32 in rank
order from +0.0 (mx/netbench.py:332-334), so all ranks end bit-identical.

Algorithms:

* ``oneshot``: K1 quantise straight into this rank's slot of the gather
  buffer -> in-place ``all_gather_into_tensor`` (N*S bytes) -> K2
  dequant-sum over the N shards -> bf16.
* ``twoshot``: K1 quantises N block-aligned chunks -> ``all_to_all_single``
  (reduce-scatter leg, 2(N-1)/N*S on the wire in total) -> K3 decodes the N
  shards of the owned chunk, sums in fp32, re-quantises -> in-place
  ``all_gather_into_tensor`` -> K2 decodes every chunk.  Requantisation adds
  at most ``block_error_bound`` per value (mx/codec.py:383-393).

The codec arithmetic lives behind a *backend* object.  The product backend
is :class:`NativeBackend` (the sm_100a kernels of libmxb200.so); the CPU
tests plug the oracle in instead to check the orchestration with ``gloo``.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

from . import _native
from .errors import MinimumDegreeTwo, NonFiniteInput, ShapeMismatch
from .formats import SchemeDescriptor, parse_scheme

ALGOS = ("oneshot", "twoshot")


def twoshot_chunk_values(n: int, nranks: int, block: int) -> int:
    """Chunk length of the two-shot path: ceil(n/N) rounded up to a multiple
    of 8*block so blocks never straddle chunks and every chunk's streams are
    byte aligned (the oracle's twoshot_chunks rule)."""
    unit = 8 * block
    per = -(-n // nranks)
    return max(unit, -(-per // unit) * unit)


def chunk_len(n: int, c: int, j: int) -> int:
    return max(0, min(c, n - j * c))


# ---------------------------------------------------------------------------
# backends
# ---------------------------------------------------------------------------


class NativeBackend:
    """Codec steps on the sm_100a kernels (stream-ordered, no host sync)."""

    def __init__(self, scheme: SchemeDescriptor):
        self.scheme = scheme
        self.cs = scheme.to_c()
        self.lib = _native.load()

    def layout(self, n: int):
        return _native.shard_layout(n, self.cs)

    def workspace(self, n: int, requant: bool = False) -> int:
        return _native.workspace_bytes(n, self.cs, requant)

    @staticmethod
    def _p(t):
        return ctypes.c_void_p(t.data_ptr())

    @staticmethod
    def _st():
        import torch

        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    @staticmethod
    def _dt(t):
        import torch

        return {torch.float32: _native.MX_F32, torch.float16: _native.MX_F16,
                torch.bfloat16: _native.MX_BF16}[t.dtype]

    def quantize_into(self, x, shard, ws, flag):
        so, eo, _ = self.layout(x.numel())
        _native.check(self.lib.mx_quantize(
            self._p(x), self._dt(x), x.numel(), ctypes.byref(self.cs),
            ctypes.c_void_p(shard.data_ptr() + so), ctypes.c_void_p(shard.data_ptr() + eo),
            self._p(flag) if flag is not None else None, self._p(ws), ws.numel(), self._st()),
            "mx_quantize")

    def quantize_chunks(self, x, c, shards, shard_stride, ws, flag):
        _native.check(self.lib.mx_quantize_chunks(
            self._p(x), self._dt(x), x.numel(), c, ctypes.byref(self.cs), self._p(shards),
            shard_stride, self._p(flag) if flag is not None else None, self._p(ws), ws.numel(),
            self._st()), "mx_quantize_chunks")

    def dequant_sum(self, shards, rank_stride, nranks, n, c, chunk_stride, out, residual=None):
        if residual is not None:  # out = residual + sum, fused into K2's store
            _native.check(self.lib.mx_dequant_sum_residual(
                self._p(shards), rank_stride, nranks, n, c, chunk_stride, ctypes.byref(self.cs),
                self._p(residual), self._p(out), self._dt(out), self._st()),
                "mx_dequant_sum_residual")
            return
        _native.check(self.lib.mx_dequant_sum(
            self._p(shards), rank_stride, nranks, n, c, chunk_stride, ctypes.byref(self.cs),
            self._p(out), self._dt(out), self._st()), "mx_dequant_sum")

    def requant(self, shards, rank_stride, nranks, n, c, out_shard, ws, flag):
        _native.check(self.lib.mx_dequant_sum_requant(
            self._p(shards), rank_stride, nranks, n, c, ctypes.byref(self.cs), self._p(out_shard),
            self._p(flag) if flag is not None else None, self._p(ws), ws.numel(), self._st()),
            "mx_dequant_sum_requant")

    def reset_flag(self, flag):
        _native.check(self.lib.mx_nonfinite_reset(self._p(flag), self._st()), "mx_nonfinite_reset")

    def gemm_supported(self, x, w) -> bool:
        """Whether the tcgen05 GEMM with the fused quantiser (k_gemm.cu)
        covers x[M, K] . w[N, K]^T under this scheme (else the caller runs
        F.linear + K1)."""
        import torch

        sch = self.scheme
        el = sch.to_c()
        fmt = (el.kind, el.exponent_bits, el.mantissa_bits)  # kind 0 float, 1 int
        B = sch.block_size
        if el.scale_bits == 8:
            ok_fmt = {32: {(0, 2, 1), (0, 2, 3), (0, 3, 2), (0, 2, 2), (1, 0, 7)},
                      16: {(0, 2, 1), (1, 0, 7)}, 8: {(0, 2, 1)}}.get(B, set())
        elif el.scale_bits == 5:  # E5M0: the paper's selected schemes, N % 256 == 0
            ok_fmt = {32: {(0, 2, 1), (0, 2, 2)}, 16: {(0, 2, 1)}, 8: {(0, 2, 1)}}.get(B, set())
            if w.dim() != 2 or w.shape[0] % 256 != 0:
                return False
        else:
            return False
        K = x.shape[-1]
        return (fmt in ok_fmt and x.dtype == torch.bfloat16
                and w.dtype == torch.bfloat16 and x.is_cuda and w.is_cuda and w.dim() == 2
                and w.shape[1] == K and K % 64 == 0 and w.shape[0] % 128 == 0
                and x.is_contiguous() and w.is_contiguous()
                and x.data_ptr() % 16 == 0 and w.data_ptr() % 16 == 0)

    def gemm_preferred(self, x, w) -> bool:
        """Whether the fused GEMM is expected to beat cuBLAS + K1 for this
        shape and scheme (measured, profiles/r02/gemm): it saves K1 (~2.5
        B/value of HBM traffic) but schedules whole 256x256 tiles over the SM
        pairs, so a badly quantised last wave costs more than K1 once the
        GEMM is long, and the quantiser in the epilogue costs more per tile
        for small blocks.  E8M0 with B in {16, 32}: fused when the tile waves
        are >= 90 % full or K <= 4096 (8B o_proj at TP=1/2 and every 8B
        projection from TP=4 win, 8B down_proj at TP=1/2 -- K = 14336 / 7168
        on 128 tiles = 1.73 waves -- loses 4-8 %).  E5M0 (the paper's
        schemes): only B = 32 with >= 90 %-full waves (fp5_e2m2:32:e5m0 at
        the 70B TP=8 shapes: 1.05-1.10x); block 8 / 16 epilogues are slower
        than cuBLAS + K1 at every measured shape (0.78-0.98x)."""
        if not self.gemm_supported(x, w):
            return False
        import torch

        K = x.shape[-1]
        M, N = x.numel() // K, w.shape[0]
        tiles = -(-M // 256) * -(-N // 256)
        pairs = max(1, torch.cuda.get_device_properties(x.device).multi_processor_count // 2)
        waves = -(-tiles // pairs)
        full = tiles / (waves * pairs) >= 0.9
        B = self.scheme.block_size
        if self.scheme.scale.exponent_bits != 8:
            return B == 32 and full
        return B >= 16 and (full or K <= 4096)

    def gemm_quantize_chunks(self, x2, w, c, shards, shard_stride, flag, partial=None):
        """k_gemm_mx: partial = x2 . w^T on the tensor cores, its MX shard(s)
        written straight from the accumulator (chunk j of c values at
        shards + j*shard_stride)."""
        M, K = x2.shape
        N = w.shape[0]
        _native.check(self.lib.mx_gemm_quantize_chunks(
            self._p(x2), self._p(w), M, N, K, c, ctypes.byref(self.cs), self._p(shards),
            shard_stride, self._p(partial) if partial is not None else None,
            self._p(flag) if flag is not None else None, self._st()), "mx_gemm_quantize_chunks")

    def allreduce_fused(self, ptrs, dtype, nranks, n, shards, stride, out, barrier, flag):
        """One persistent kernel: quantise the local partials, grid barrier,
        dequant-sum.  Returns False when the scheme/dtype has no fused
        instantiation (the caller then runs K1 + K2)."""
        rc = self.lib.mx_allreduce_fused(
            self._p(ptrs), dtype, nranks, n, ctypes.byref(self.cs), self._p(shards), stride,
            self._p(out), self._dt(out), self._p(barrier),
            self._p(flag) if flag is not None else None, self._st())
        if rc == -8:  # MX_ERR_UNSUPPORTED
            return False
        _native.check(rc, "mx_allreduce_fused")
        return True


# ---------------------------------------------------------------------------
# the collective
# ---------------------------------------------------------------------------


@dataclass
class _Plan:
    n: int
    nranks: int
    algo: str
    shard_bytes: int  # one-shot: S(n); two-shot: S(c)
    c: int            # two-shot chunk values (n for one-shot)


class CompressedAllReduce:
    """Persistent-buffer compressed all-reduce of an ``n``-value activation.

    ``out = car(x)`` reduces the row-parallel partial ``x`` (bf16/f16/f32
    CUDA tensor, any shape with ``n`` values) across ``group`` and returns
    the sum in ``out_dtype``.  Buffers are allocated once, so the call is
    CUDA-graph capturable (NCCL collectives capture).  Non-finite inputs are
    recorded in a sticky device flag; :meth:`check_finite` raises
    NonFiniteInput later (deferred, no sync on the hot path).
    """

    def __init__(self, scheme, n: int, group=None, algo: str = "oneshot", out_dtype=None,
                 device=None, backend=None, world_size: int | None = None,
                 rank: int | None = None, comm=None):
        import torch
        import torch.distributed as dist

        if isinstance(scheme, str):
            scheme = parse_scheme(scheme, extensions=True)
        if algo not in ALGOS:
            raise ValueError(f"algo must be one of {ALGOS}")
        self.scheme = scheme
        self.group = group
        # the exchange: torch.distributed (NCCL; gloo in the CPU tests) once a
        # process group exists -- at every world size, so a world-1 NCCL run
        # issues the same collectives as TP=N -- or any object with the same
        # all_gather_into_tensor / all_to_all_single (LocalThreadGroup: N
        # ranks as N threads on one GPU)
        if comm is None and dist.is_available() and dist.is_initialized():
            comm = dist
        self.comm = comm
        if comm is None or comm is dist:
            self.world = world_size if world_size is not None else (
                dist.get_world_size(group) if comm is not None else 1)
            self.rank = rank if rank is not None else (
                dist.get_rank(group) if comm is not None else 0)
        else:
            self.world = world_size if world_size is not None else comm.get_world_size()
            self.rank = rank if rank is not None else comm.get_rank()
        if self.world < 1:
            raise MinimumDegreeTwo("world size must be positive")
        if self.world > 1 and comm is None:
            raise MinimumDegreeTwo("world size > 1 needs a process group or a comm object")
        if not 0 <= self.rank < self.world:
            raise ValueError(f"rank {self.rank} outside world size {self.world}")
        self.algo = algo
        self.n = int(n)
        self.out_dtype = out_dtype or torch.bfloat16
        self.device = torch.device(device) if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available()
            else torch.device("cpu"))
        self.backend = backend or NativeBackend(scheme)
        B = scheme.block_size
        N = self.world
        if algo == "oneshot":
            c = self.n
            _, _, S = self.backend.layout(self.n)
            self.gathered = torch.empty(N * S, dtype=torch.uint8, device=self.device)
            self.ws = torch.empty(self.backend.workspace(self.n), dtype=torch.uint8,
                                  device=self.device)
        else:
            c = twoshot_chunk_values(self.n, N, B)
            _, _, S = self.backend.layout(c)
            self.send = torch.empty(N * S, dtype=torch.uint8, device=self.device)
            self.recv = torch.empty(N * S, dtype=torch.uint8, device=self.device)
            self.gathered = torch.empty(N * S, dtype=torch.uint8, device=self.device)
            self.ws = torch.empty(max(self.backend.workspace(N * c),
                                      self.backend.workspace(c, requant=True)),
                                  dtype=torch.uint8, device=self.device)
        self.plan = _Plan(self.n, N, algo, S, c)
        self.flag = torch.empty(1, dtype=torch.int64, device=self.device)
        self.backend.reset_flag(self.flag)
        self.out = torch.empty(self.n, dtype=self.out_dtype, device=self.device)

    # -- wire accounting ----------------------------------------------------
    @property
    def wire_bytes_per_rank(self) -> int:
        """Bytes this rank sends (= receives) per call."""
        N, S = self.plan.nranks, self.plan.shard_bytes
        return (N - 1) * S if self.algo == "oneshot" else 2 * (N - 1) * S

    def _check_residual(self, residual):
        if residual is None:
            return None
        if residual.numel() != self.n or residual.dtype != self.out_dtype or \
                not residual.is_contiguous():
            raise ShapeMismatch(f"residual must be a contiguous {self.out_dtype} tensor of "
                                f"{self.n} values")
        return residual.reshape(-1)

    def __call__(self, x, out=None, residual=None):
        """all_reduce(x); with ``residual`` the result is ``residual +
        all_reduce(x)`` computed in K2's store (bit-identical to the unfused
        add in out_dtype; ``out`` may be ``residual`` for an in-place update)."""
        if x.numel() != self.n:
            raise ShapeMismatch(f"expected {self.n} values, got {x.numel()}")
        out = self._reduce(x.reshape(-1), None, out, self._check_residual(residual))
        return out.view(x.shape) if out.numel() == x.numel() else out

    def linear(self, x, weight, out=None, residual=None):
        """all_reduce(F.linear(x, weight)) -- the row-parallel hook
        (mx/tpsim.py:263-265) with the quantiser fused into the GEMM
        epilogue (k_gemm.cu, tcgen05 + TMA): the bf16 partial is never
        written; the shard comes straight out of the accumulator, then the
        exchange and dequant-sum run as in __call__.  Falls back to
        F.linear + __call__ where the fused GEMM does not apply."""
        import torch.nn.functional as F

        K = x.shape[-1]
        N = weight.shape[0]
        M = x.numel() // K if K else 0
        if M * N != self.n:
            raise ShapeMismatch(f"expected {self.n} output values, got {M}x{N}")
        be = self.backend
        if not (hasattr(be, "gemm_supported") and be.gemm_supported(x, weight)):
            return self(F.linear(x, weight), out, residual)
        res = self._reduce(None, (x.reshape(M, K), weight), out, self._check_residual(residual))
        return res.view(*x.shape[:-1], N)

    def _reduce(self, xf, gemm, out, residual=None):
        out = self.out if out is None else out.reshape(-1)
        p, be, N, comm = self.plan, self.backend, self.plan.nranks, self.comm
        S = p.shard_bytes
        if self.algo == "oneshot":
            mine = self.gathered[self.rank * S:(self.rank + 1) * S]
            if gemm is None:
                be.quantize_into(xf, mine, self.ws, self.flag)
            else:
                be.gemm_quantize_chunks(gemm[0], gemm[1], p.n, mine, S, self.flag)
            if comm is not None:
                comm.all_gather_into_tensor(self.gathered, mine, group=self.group)
            if residual is None:
                be.dequant_sum(self.gathered, S, N, p.n, p.n, 0, out)
            else:
                be.dequant_sum(self.gathered, S, N, p.n, p.n, 0, out, residual)
        else:
            if gemm is None:
                be.quantize_chunks(xf, p.c, self.send, S, self.ws, self.flag)
            else:
                be.gemm_quantize_chunks(gemm[0], gemm[1], p.c, self.send, S, self.flag)
            if comm is not None:
                comm.all_to_all_single(self.recv, self.send, group=self.group)
                recv = self.recv
            else:
                recv = self.send
            mine = self.gathered[self.rank * S:(self.rank + 1) * S]
            own = chunk_len(p.n, p.c, self.rank)
            if own > 0:
                be.requant(recv, S, N, own, p.c, mine, self.ws, self.flag)
            if comm is not None:
                comm.all_gather_into_tensor(self.gathered, mine, group=self.group)
            if residual is None:
                be.dequant_sum(self.gathered, 0, 1, p.n, p.c, S, out)
            else:
                be.dequant_sum(self.gathered, 0, 1, p.n, p.c, S, out, residual)
        return out

    def check_finite(self):
        """Raise NonFiniteInput if any call since the last check saw NaN/Inf.
        The flag holds the first flat index in this rank's partial (both
        algorithms: K1 reports it; non-finite blocks are zeroed before the
        exchange), so block_index = index // B as in _check_finite
        (mx/codec.py:191-199)."""
        idx = int(self.flag.item())
        if idx >= 0:
            self.backend.reset_flag(self.flag)
            raise NonFiniteInput(f"non-finite value in a compressed all-reduce input "
                                 f"(flat index {idx})",
                                 block_index=idx // self.scheme.block_size)

    def check_status(self):
        """NCCL reports its own failures; nothing to poll (API parity with
        SymmetricAllReduce)."""


def compressed_all_reduce(x, scheme, group=None, algo: str = "oneshot", out_dtype=None):
    """One-off convenience wrapper (allocates buffers per call)."""
    car = CompressedAllReduce(scheme, x.numel(), group=group, algo=algo,
                              out_dtype=out_dtype or x.dtype, device=x.device)
    return car(x).clone()


# ---------------------------------------------------------------------------
# fused over symmetric memory (NVLink pull), one kernel per rank per call
# ---------------------------------------------------------------------------


class SymmetricAllReduce:
    """One-shot compressed all-reduce fused into ONE kernel per rank over
    torch symmetric memory (peer-mapped buffers on NVLink / NVSwitch).

    Per-CTA dataflow (k_symm_flow): CTA b of every rank quantises the same
    8 units of its partial into its own shard slot, raises a system-scope
    flag for CTA b in every peer's flag array, waits for the N flags of CTA
    b and decodes those units of all N shards straight out of the peers'
    memory, in rank order, into fp32 -> ``out_dtype``.  This replaces K1 ->
    NCCL all-gather -> K2 (mx/netbench.py:323-334) with no gather buffer, no
    NCCL kernel and no grid-wide barrier; the result is bit-identical to the
    NCCL one-shot (same codes, same sum order).  A peer wait longer than
    ~2 s sets a status word instead of hanging (:meth:`check_status`).
    ``algo="twoshot"`` runs k_symm2_flow instead (the TP >= 4 algorithm:
    reduce-scatter leg as peer pulls of this rank's chunk, fp32 sum and
    re-quantisation, then pulls of every owner's reduced chunk), bit-identical
    to the NCCL two-shot.
    Requirements: bf16 partial, n % 1024 == 0 (two-shot: n % (1024*N) == 0),
    B in {16,32,64} (any scale width: E8M0, E5M0, ...).
    """

    def __init__(self, scheme, n: int, group=None, out_dtype=None, device=None,
                 algo: str = "oneshot"):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem

        if isinstance(scheme, str):
            scheme = parse_scheme(scheme, extensions=True)
        if algo not in ALGOS:
            raise ValueError(f"algo must be one of {ALGOS}")
        self.scheme, self.n, self.algo = scheme, int(n), algo
        self.group = group or dist.group.WORLD
        self.world = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self.out_dtype = out_dtype or torch.bfloat16
        self.backend = NativeBackend(scheme)
        if algo == "oneshot":
            self.slot, flags_off, total, ctas = _native.symm_layout(self.n, self.backend.cs,
                                                                    self.world)
        else:  # k_symm2_flow: n % (1024 * world) == 0
            self.slot, _, flags_off, total, ctas = _native.symm_twoshot_layout(
                self.n, self.backend.cs, self.world)
        self.buf = symm_mem.empty(total, dtype=torch.uint8, device=self.device)
        self.hdl = symm_mem.rendezvous(self.buf, self.group)
        # flags start at zero on every rank before anyone can signal
        self.buf[flags_off:].zero_()
        self.flag_ptrs = torch.tensor([int(p) + flags_off for p in self.hdl.buffer_ptrs],
                                      dtype=torch.int64, device=self.device)
        torch.cuda.synchronize()
        dist.barrier(self.group)
        self.state = torch.zeros(1 + ctas, dtype=torch.int32, device=self.device)  # status, epochs
        self.flag = torch.empty(1, dtype=torch.int64, device=self.device)
        self.backend.reset_flag(self.flag)
        self.out = torch.empty(self.n, dtype=self.out_dtype, device=self.device)

    def __call__(self, x, out=None, residual=None):
        """all_reduce(x), or ``residual + all_reduce(x)`` fused into the
        kernel's store (as CompressedAllReduce.__call__)."""
        import torch

        if x.numel() != self.n or x.dtype != torch.bfloat16 or not x.is_contiguous():
            raise ShapeMismatch(f"expected a contiguous bf16 tensor of {self.n} values")
        if residual is not None and (residual.numel() != self.n or
                                     residual.dtype != self.out_dtype or
                                     not residual.is_contiguous()):
            raise ShapeMismatch(f"residual must be a contiguous {self.out_dtype} tensor of "
                                f"{self.n} values")
        res = ctypes.c_void_p(residual.data_ptr()) if residual is not None else None
        o = self.out if out is None else out.reshape(-1)
        be = self.backend
        base = self.state.data_ptr()
        if self.algo == "oneshot":
            rc = be.lib.mx_allreduce_symm(
                ctypes.c_void_p(x.data_ptr()), _native.MX_BF16, self.n, ctypes.byref(be.cs),
                ctypes.c_void_p(self.hdl.buffer_ptrs_dev),
                ctypes.c_void_p(self.flag_ptrs.data_ptr()), self.rank, self.world, self.slot,
                ctypes.c_void_p(o.data_ptr()), be._dt(o), res, ctypes.c_void_p(base),
                ctypes.c_void_p(base + 4), ctypes.c_void_p(self.flag.data_ptr()), be._st())
        else:
            rc = be.lib.mx_allreduce_symm_twoshot(
                ctypes.c_void_p(x.data_ptr()), _native.MX_BF16, self.n, ctypes.byref(be.cs),
                ctypes.c_void_p(self.hdl.buffer_ptrs_dev),
                ctypes.c_void_p(self.flag_ptrs.data_ptr()), self.rank, self.world,
                ctypes.c_void_p(o.data_ptr()), be._dt(o), res, ctypes.c_void_p(base),
                ctypes.c_void_p(base + 4), ctypes.c_void_p(self.flag.data_ptr()), be._st())
        _native.check(rc, "mx_allreduce_symm")
        return o.view(x.shape)

    def check_status(self):
        """Raise if a peer wait timed out (the results of that call are invalid)."""
        if int(self.state[0].item()) != 0:
            raise RuntimeError("symmetric-memory all-reduce: a peer flag wait timed out")

    def check_finite(self):
        idx = int(self.flag.item())
        if idx >= 0:
            self.backend.reset_flag(self.flag)
            raise NonFiniteInput(f"non-finite value in a compressed all-reduce input "
                                 f"(flat index {idx})", block_index=idx // self.scheme.block_size)


# ---------------------------------------------------------------------------
# N ranks as N host threads on ONE device (the in-process transport)
# ---------------------------------------------------------------------------


def push_scheme_ok(sch) -> bool:
    """The GEMM push's scheme set (k_gemm.cu launch_gemm_mx_push, k_push.cu
    MXB_PUSH_SET): fp4_e2m1 E8M0 B 16/32 and the paper's E5M0 schemes --
    fp4_e2m1 B 8/16/32, fp5_e2m2 B 32."""
    e, k, b = sch.element.name, sch.scale.exponent_bits, sch.block_size
    if k == 8:
        return e == "fp4_e2m1" and b in (16, 32)
    if k == 5:
        return (e == "fp4_e2m1" and b in (8, 16, 32)) or (e == "fp5_e2m2" and b == 32)
    return False


class FusedLinearAllReduce:
    """all_reduce(x @ W^T) with the GEMM, the MX quantiser AND the all-gather
    in ONE kernel per rank, over torch symmetric memory (NVLink / NVSwitch).

    The tcgen05 row-parallel GEMM (k_gemm.cu, 2-CTA form) quantises each
    accumulator tile as it drains and stores the shard bytes straight into
    slot (epoch & 1) of every rank's symmetric buffer -- the all-gather of
    mx/netbench.py:323-328 rides on the epilogue and overlaps the remaining
    tiles' math; its last CTA (GPU-scope arrival counter) issues one
    system-scope fence and publishes the epoch into every rank's flag array.
    A second launch (k_push_dqsum) waits for the N flags and decodes the N
    shards from local memory in rank order, with the optional residual add
    fused into its store.  Bit-identical to ``CompressedAllReduce.linear``
    (NCCL one-shot) on the same operands.  No NCCL kernel, no gather copy.
    ``algo="twoshot"`` (TP >= 4): the epilogue scatters chunk j of the shard
    to rank j only (the reduce-scatter leg rides on the GEMM); a requantise
    launch waits for the N chunks, sums this rank's chunk over the senders in
    rank order, re-quantises it and pushes it into every rank (the
    all-gather leg, published by its last CTA); the decode launch waits and
    decodes every owner's chunk -- bit-identical to the NCCL two-shot
    (n % (1024 * world) == 0).
    Requirements: a scheme of the push set (``push_scheme_ok``: fp4_e2m1
    E8M0 with B in {16, 32}, the paper's fp4_e2m1 E5M0 with B in {8, 16, 32}
    and fp5_e2m2 E5M0 with B = 32); bf16 x [M, K] and
    W [N, K] contiguous, N % 256 == 0, K % 64 == 0, n = M*N % 1024 == 0;
    at most 8 ranks.  Slots alternate by epoch parity, which is safe because a
    rank starts call e only after its call e-1 saw every peer's e-1 flag,
    i.e. after every peer finished reading slot (e & 1) in call e-2.
    """

    def __init__(self, scheme, n: int, group=None, out_dtype=None, device=None,
                 algo: str = "oneshot"):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem

        if isinstance(scheme, str):
            scheme = parse_scheme(scheme, extensions=True)
        self.scheme, self.n = scheme, int(n)
        self.group = group or dist.group.WORLD
        self.world = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)
        if self.world > 8:
            raise ShapeMismatch("the GEMM + all-gather push supports at most 8 ranks")
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self.out_dtype = out_dtype or torch.bfloat16
        self.backend = NativeBackend(scheme)
        if algo not in ("oneshot", "twoshot"):
            raise ValueError("algo must be 'oneshot' or 'twoshot'")
        self.algo = algo
        if algo == "oneshot":
            self.slot, self.shard_stride, flags_off, total = _native.push_layout(
                self.n, self.backend.cs, self.world)
        else:
            _c, self.slot, self.shard_stride, flags_off, total = _native.push2_layout(
                self.n, self.backend.cs, self.world)
        self.buf = symm_mem.empty(total, dtype=torch.uint8, device=self.device)
        self.hdl = symm_mem.rendezvous(self.buf, self.group)
        self.buf[flags_off:].zero_()  # flags start at zero before anyone can signal
        self.flags_local = self.buf[flags_off:]
        self.buf_ptrs = torch.tensor([int(p) for p in self.hdl.buffer_ptrs], dtype=torch.int64,
                                     device=self.device)
        self.flag_ptrs = torch.tensor([int(p) + flags_off for p in self.hdl.buffer_ptrs],
                                      dtype=torch.int64, device=self.device)
        torch.cuda.synchronize()
        dist.barrier(self.group)
        # [0] status (as SymmetricAllReduce), [1] epoch, [2] GEMM CTA counter,
        # [3] two-shot requantiser CTA counter
        self.state = torch.zeros(4, dtype=torch.int32, device=self.device)
        self.flag = torch.empty(1, dtype=torch.int64, device=self.device)
        self.backend.reset_flag(self.flag)
        self.out = torch.empty(self.n, dtype=self.out_dtype, device=self.device)

    def supported(self, x, w) -> bool:
        import torch

        sch = self.scheme
        return (push_scheme_ok(sch) and x.dtype == torch.bfloat16
                and (self.algo == "oneshot" or self.n % (1024 * self.world) == 0)
                and w.dtype == torch.bfloat16 and w.dim() == 2 and x.shape[-1] == w.shape[1]
                and w.shape[0] % 256 == 0 and x.shape[-1] % 64 == 0 and self.n % 1024 == 0
                and x.is_contiguous() and w.is_contiguous()
                and x.numel() // x.shape[-1] * w.shape[0] == self.n)

    def linear(self, x, weight, out=None, residual=None):
        """all_reduce(F.linear(x, weight)) [+ residual], two launches per rank."""
        import torch

        if not self.supported(x, weight):
            raise ShapeMismatch("FusedLinearAllReduce: unsupported operands for the push GEMM")
        if residual is not None and (residual.numel() != self.n or
                                     residual.dtype != self.out_dtype or
                                     not residual.is_contiguous()):
            raise ShapeMismatch(f"residual must be a contiguous {self.out_dtype} tensor of "
                                f"{self.n} values")
        K = x.shape[-1]
        M, N = x.numel() // K, weight.shape[0]
        o = self.out if out is None else out.reshape(-1)
        be = self.backend
        P = ctypes.c_void_p
        base = self.state.data_ptr()
        res = P(residual.data_ptr()) if residual is not None else None
        if self.algo == "twoshot":
            _native.check(be.lib.mx_gemm_reducescatter_push(
                P(x.data_ptr()), P(weight.data_ptr()), M, N, K, ctypes.byref(be.cs),
                P(self.buf_ptrs.data_ptr()), self.rank, self.world, P(base + 4),
                P(self.flag.data_ptr()), be._st()), "mx_gemm_reducescatter_push")
            _native.check(be.lib.mx_push2_requant(
                P(self.buf.data_ptr()), self.n, ctypes.byref(be.cs), self.rank, self.world,
                P(self.buf_ptrs.data_ptr()), P(self.flag_ptrs.data_ptr()), P(base + 4), P(base),
                P(self.flag.data_ptr()), be._st()), "mx_push2_requant")
            _native.check(be.lib.mx_push2_decode(
                P(self.buf.data_ptr()), self.n, ctypes.byref(be.cs), self.rank, self.world,
                P(base + 4), P(base), P(o.data_ptr()), be._dt(o), res, be._st()),
                "mx_push2_decode")
            return o.view(*x.shape[:-1], N)
        _native.check(be.lib.mx_gemm_allgather_push(
            P(x.data_ptr()), P(weight.data_ptr()), M, N, K, ctypes.byref(be.cs),
            P(self.buf_ptrs.data_ptr()), self.rank, self.world,
            P(base + 4), P(self.flag.data_ptr()), be._st()), "mx_gemm_allgather_push")
        _native.check(be.lib.mx_push_dequant_sum(
            P(self.buf.data_ptr()), self.n, ctypes.byref(be.cs), self.rank, self.world,
            P(self.flags_local.data_ptr()), P(base + 4), P(base), P(o.data_ptr()), be._dt(o),
            P(residual.data_ptr()) if residual is not None else None, be._st()),
            "mx_push_dequant_sum")
        return o.view(*x.shape[:-1], N)

    def check_status(self):
        """Raise if a peer wait timed out (the results of that call are invalid)."""
        if int(self.state[0].item()) != 0:
            raise RuntimeError("GEMM + all-gather push: a peer flag wait timed out")

    def check_finite(self):
        idx = int(self.flag.item())
        if idx >= 0:
            self.backend.reset_flag(self.flag)
            raise NonFiniteInput(f"non-finite value in a row-parallel partial (flat index {idx})",
                                 block_index=idx // self.scheme.block_size)


class LocalThreadGroup:
    """A process-group stand-in for N ranks that are N host threads sharing
    one GPU -- the device form of the reference's in-process mailbox
    transport (mx/netbench.py:186-203, N worker threads).

    Each rank thread calls :meth:`bind` once and issues its work on its own
    CUDA stream.  ``all_gather_into_tensor`` / ``all_to_all_single`` have
    the torch.distributed signatures and semantics: every rank's input is
    read after that rank's preceding work (CUDA events), the placement is a
    stream-ordered device copy, and no rank proceeds (on the device) past
    the collective until every peer has read its input -- so
    :class:`CompressedAllReduce` runs its real NCCL code path, with the real
    kernels, at any N on one GPU."""

    def __init__(self, world_size: int, device=None, timeout: float = 120.0):
        import threading

        import torch

        if world_size < 1:
            raise MinimumDegreeTwo("world size must be positive")
        self.world = int(world_size)
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self._tls = threading.local()
        self._barrier = threading.Barrier(self.world, timeout=timeout)
        self._slots = [None] * self.world
        self._done = [None] * self.world

    def bind(self, rank: int) -> None:
        if not 0 <= rank < self.world:
            raise ValueError(f"rank {rank} outside world size {self.world}")
        self._tls.rank = rank

    def get_rank(self, group=None) -> int:
        return self._tls.rank

    def get_world_size(self, group=None) -> int:
        return self.world

    def abort(self) -> None:
        self._barrier.abort()

    def _exchange(self, out, inp, place) -> None:
        import torch

        r = self._tls.rank
        st = torch.cuda.current_stream(self.device)
        ready = torch.cuda.Event()
        ready.record(st)
        self._slots[r] = (inp, ready)
        self._barrier.wait()
        for j in range(self.world):
            src, ev = self._slots[j]
            st.wait_event(ev)
            place(j, src)
        done = torch.cuda.Event()
        done.record(st)
        self._done[r] = done
        self._barrier.wait()
        for j in range(self.world):  # every peer has read my input
            st.wait_event(self._done[j])

    def all_gather_into_tensor(self, out, inp, group=None, async_op=False):
        S = inp.numel()
        if out.numel() != S * self.world:
            raise ShapeMismatch("all_gather_into_tensor: output must hold world x input")

        def place(j, src):
            dst = out[j * S:(j + 1) * S]
            if dst.data_ptr() != src.data_ptr():
                dst.copy_(src, non_blocking=True)

        self._exchange(out, inp, place)

    def all_to_all_single(self, out, inp, group=None, async_op=False):
        S = inp.numel() // self.world
        if inp.numel() != S * self.world or out.numel() != inp.numel():
            raise ShapeMismatch("all_to_all_single: equal splits of world chunks")
        r = self._tls.rank

        def place(j, src):
            out[j * S:(j + 1) * S].copy_(src[r * S:(r + 1) * S], non_blocking=True)

        self._exchange(out, inp, place)

    def run(self, fn):
        """Run ``fn(rank)`` on one thread per rank, each bound to its rank
        and its own stream; returns the results in rank order and re-raises
        the first failure (the barrier is aborted so no thread hangs)."""
        import threading

        import torch

        res = [None] * self.world
        errs = []

        def work(r):
            try:
                torch.cuda.set_device(self.device)
                self.bind(r)
                with torch.cuda.stream(torch.cuda.Stream(self.device)):
                    res[r] = fn(r)
                    torch.cuda.current_stream(self.device).synchronize()
            except threading.BrokenBarrierError as e:
                errs.append((r, e))
            except BaseException as e:  # noqa: BLE001
                errs.append((r, e))
                self._barrier.abort()

        ts = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(self.world)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        if errs:
            root = next((e for r, e in errs if not isinstance(e, threading.BrokenBarrierError)),
                        errs[0][1])
            self._barrier.reset()
            raise root
        return res


# ---------------------------------------------------------------------------
# single-GPU simulation of N ranks (same kernels, exchange = buffer copies)
# ---------------------------------------------------------------------------


class SimulatedAllReduce:
    """N TP ranks on ONE device: the same K1/K2/K3 kernels as
    :class:`CompressedAllReduce`, with the NCCL exchange replaced by the
    equivalent buffer placement (one-shot: every rank quantises straight into
    its slot of the gathered buffer; two-shot: the all-to-all is a strided
    copy).  Persistent buffers, so a call is CUDA-graph capturable.  This is
    the single-GPU parity harness and the N=1 bench workload ("simulated
    TP=2", BASELINE.json configs[0])."""

    def __init__(self, scheme, n: int, nranks: int, algo: str = "oneshot", out_dtype=None,
                 device="cuda", backend=None, fused: bool = True):
        import torch

        if isinstance(scheme, str):
            scheme = parse_scheme(scheme, extensions=True)
        if algo not in ALGOS:
            raise ValueError(f"algo must be one of {ALGOS}")
        self.scheme, self.n, self.N, self.algo = scheme, int(n), int(nranks), algo
        self.be = backend or NativeBackend(scheme)
        self.device = torch.device(device)
        self.out_dtype = out_dtype or torch.bfloat16
        N, n = self.N, self.n
        dev = self.device
        self.flag = torch.empty(1, dtype=torch.int64, device=dev)
        self.be.reset_flag(self.flag)
        self.out = torch.empty(n, dtype=self.out_dtype, device=dev)
        # fused one-shot (one persistent kernel) when the backend offers it
        import os

        self.fused = (fused and algo == "oneshot" and hasattr(self.be, "allreduce_fused")
                      and os.environ.get("MXB200_FUSED", "1") != "0")
        self._ptrs_key = None
        self.barrier = torch.zeros(2, dtype=torch.int32, device=dev) if self.fused else None
        if algo == "oneshot":
            _, _, S = self.be.layout(n)
            self.S, self.c = S, n
            self.gathered = torch.empty(N * S, dtype=torch.uint8, device=dev)
            self.ws = torch.empty(self.be.workspace(n), dtype=torch.uint8, device=dev)
        else:
            self.c = twoshot_chunk_values(n, N, scheme.block_size)
            _, _, S = self.be.layout(self.c)
            self.S = S
            self.send = torch.empty(N, N * S, dtype=torch.uint8, device=dev)
            self.recv = torch.empty(N, N * S, dtype=torch.uint8, device=dev)
            self.gathered = torch.empty(N * S, dtype=torch.uint8, device=dev)
            self.ws = torch.empty(max(self.be.workspace(N * self.c),
                                      self.be.workspace(self.c, requant=True)),
                                  dtype=torch.uint8, device=dev)

    @property
    def shard_bytes(self) -> int:
        return self.S

    def quantize(self, partials):
        """K1 for every rank (one-shot: into the gathered buffer)."""
        be, S = self.be, self.S
        if self.algo == "oneshot":
            for r, p in enumerate(partials):
                be.quantize_into(p.reshape(-1), self.gathered[r * S:(r + 1) * S], self.ws,
                                 self.flag)
        else:
            for r, p in enumerate(partials):
                be.quantize_chunks(p.reshape(-1), self.c, self.send[r], S, self.ws, self.flag)

    def reduce(self, out=None):
        """Everything after K1: (exchange) + K3 + K2."""
        be, S, N, n, c = self.be, self.S, self.N, self.n, self.c
        out = self.out if out is None else out.reshape(-1)
        if self.algo == "oneshot":
            be.dequant_sum(self.gathered, S, N, n, n, 0, out)
        else:
            # all-to-all: owner j receives chunk j of every rank, in rank order
            self.recv.view(N, N, S).copy_(self.send.view(N, N, S).transpose(0, 1))
            for j in range(N):
                own = chunk_len(n, c, j)
                if own > 0:
                    be.requant(self.recv[j], S, N, own, c, self.gathered[j * S:(j + 1) * S],
                               self.ws, self.flag)
            be.dequant_sum(self.gathered, 0, 1, n, c, S, out)
        return out

    def __call__(self, partials, out=None):
        if len(partials) != self.N or any(p.numel() != self.n for p in partials):
            raise ShapeMismatch(f"expected {self.N} partials of {self.n} values")
        if self.fused and self._fused(partials, out):
            return (self.out if out is None else out).view(partials[0].shape)
        self.quantize(partials)
        return self.reduce(out).view(partials[0].shape)

    def _fused(self, partials, out):
        import torch

        if any(p.dtype != torch.bfloat16 or not p.is_contiguous() for p in partials):
            return False
        key = tuple(p.data_ptr() for p in partials)
        if key != self._ptrs_key:  # device array of the partials' addresses
            self._ptrs = torch.tensor(key, dtype=torch.int64).to(self.device)
            self._ptrs_key = key
        o = self.out if out is None else out.reshape(-1)
        ok = self.be.allreduce_fused(self._ptrs, _native.MX_BF16, self.N, self.n, self.gathered,
                                     self.S, o, self.barrier, self.flag)
        if not ok:
            self.fused = False
        return ok


class HostPipeline:
    """Compressed all-reduce of HOST-resident partial sums into a host
    buffer -- the shape of the reference's own API, whose codec takes and
    returns host arrays (``compress_tensor(np.ndarray)`` mx/codec.py:238,
    ``decompress_tensor`` mx/codec.py:266, the exchange of
    mx/netbench.py:323-334).

    The flat tensor is cut into pieces whose lengths are multiples of 1024
    values (``chunks`` equal pieces, or a tuple of piece weights such as
    ``(1, 3, 3, 1)`` whose small head and tail pieces shorten the parts of
    the transfer that cannot overlap), so no MX block straddles a piece and
    every value's reduction is identical to the whole-tensor call.  Piece j's
    pinned host->device copies, its compressed all-reduce (one persistent
    op per piece, so its device pointers stay fixed) and its device->host
    copy are issued on three streams ordered by events: the PCIe traffic in
    both directions overlaps the kernels of neighbouring pieces.

    ``make_op(c)`` returns a callable ``(device_inputs, device_out) -> out``
    reducing ``c`` values, e.g. a :class:`SimulatedAllReduce` (all ranks'
    partials on one GPU) or a :class:`CompressedAllReduce` (this rank's
    partial, NCCL exchange).
    """

    MAX_GRAPHS = 8  # captured host-buffer sets kept (LRU)

    def __init__(self, make_op, n: int, ninputs: int, in_dtype=None, out_dtype=None,
                 device="cuda", chunks=4, graph: bool = True, h2d_streams: int = 1,
                 collective: bool = False):
        import torch

        self.n, self.nin = int(n), int(ninputs)
        self.use_graph = graph
        # ops holding NCCL collectives: a graph-cache miss captures WITHOUT
        # an eager warm-up issue, so every call runs each collective exactly
        # once whether this rank hit or missed its (rank-local) graph cache
        # and whether its host buffers were pinned -- ranks can never issue
        # different numbers of collectives
        self.collective = bool(collective)
        self._graphs = {}
        if isinstance(chunks, (list, tuple)):
            # explicit piece weights, e.g. (1, 3, 3, 1): small first and last
            # pieces shorten the un-overlapped head (H2D) and tail (D2H)
            units, tot = self.n // 1024, float(sum(chunks))
            cuts = [0]
            for wgt in chunks[:-1]:
                cuts.append(min(units, cuts[-1] + max(1, round(units * wgt / tot))))
            cuts.append(units)
            bounds = [c * 1024 for c in cuts]
            if self.n % 1024 or any(b1 <= b0 for b0, b1 in zip(bounds, bounds[1:])):
                bounds = [0, self.n]
        else:
            k = max(1, int(chunks))
            while k > 1 and (self.n % k or (self.n // k) % 1024):
                k -= 1
            bounds = [j * (self.n // k) for j in range(k + 1)]
        self.bounds = bounds
        self.k = len(bounds) - 1
        self.c = bounds[1] - bounds[0]
        self.device = torch.device(device)
        in_dtype = in_dtype or torch.bfloat16
        self.out_dtype = out_dtype or torch.bfloat16
        self.ops = [make_op(b1 - b0) for b0, b1 in zip(bounds, bounds[1:])]
        k = self.k
        self.dev_in = [torch.empty(self.n, dtype=in_dtype, device=self.device)
                       for _ in range(self.nin)]
        self.dev_out = torch.empty(self.n, dtype=self.out_dtype, device=self.device)
        # [reduce, device->host, host->device x h2d_streams]
        self.streams = [torch.cuda.Stream(self.device) for _ in range(2 + max(1, h2d_streams))]
        self.ev_in = [[torch.cuda.Event() for _ in range(self.nin)] for _ in range(k)]
        self.ev_red = [torch.cuda.Event() for _ in range(k)]

    @property
    def h2d_bytes(self) -> int:
        return self.nin * self.n * self.dev_in[0].element_size()

    @property
    def d2h_bytes(self) -> int:
        return self.n * self.dev_out.element_size()

    def __call__(self, host_inputs, host_out):
        """Run the whole pipeline; ``host_out`` is complete once the current
        stream reaches this point (e.g. after a synchronize).

        The 3k copies and k all-reduces are captured once per (host buffer
        set) into a CUDA graph with the three streams as parallel branches,
        so a call costs one graph launch instead of ~4k host-side issues
        (eager issue is host-bound: tens of microseconds per piece)."""
        import torch

        if len(host_inputs) != self.nin or any(h.numel() != self.n for h in host_inputs):
            raise ShapeMismatch(f"expected {self.nin} host tensors of {self.n} values")
        if host_out.numel() != self.n:
            raise ShapeMismatch(f"host_out must hold {self.n} values")
        hin = [h.reshape(-1) for h in host_inputs]
        hout = host_out.reshape(-1)
        pinned = all(h.is_pinned() for h in hin) and hout.is_pinned()
        if not (self.use_graph and pinned):
            self._issue(hin, hout)
            return host_out
        key = tuple(h.data_ptr() for h in hin) + (hout.data_ptr(),)
        g = self._graphs.pop(key, None)
        if g is None:
            if not self.collective:
                self._issue(hin, hout)  # first-call allocations happen eagerly
            torch.cuda.synchronize(self.device)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._issue(hin, hout)
            while len(self._graphs) >= self.MAX_GRAPHS:  # least recently used out
                self._graphs.pop(next(iter(self._graphs)))
        self._graphs[key] = g  # (re)inserted last: most recently used
        g.replay()
        return host_out

    def _issue(self, hin, hout):
        import torch

        cur = torch.cuda.current_stream(self.device)
        s_red, s_out, s_ins = self.streams[0], self.streams[1], self.streams[2:]
        for s in self.streams:
            s.wait_stream(cur)
        for j in range(self.k):
            sl = slice(self.bounds[j], self.bounds[j + 1])
            for i, (d, h) in enumerate(zip(self.dev_in, hin)):
                s_in = s_ins[i % len(s_ins)]
                with torch.cuda.stream(s_in):
                    d[sl].copy_(h[sl], non_blocking=True)
                    self.ev_in[j][i].record(s_in)
            with torch.cuda.stream(s_red):
                for i in range(self.nin):
                    s_red.wait_event(self.ev_in[j][i])
                self.ops[j]([d[sl] for d in self.dev_in], self.dev_out[sl])
                self.ev_red[j].record(s_red)
            with torch.cuda.stream(s_out):
                s_out.wait_event(self.ev_red[j])
                hout[sl].copy_(self.dev_out[sl], non_blocking=True)
        for s in self.streams:
            cur.wait_stream(s)

    @classmethod
    def simulated(cls, scheme, n: int, nranks: int, algo: str = "oneshot", out_dtype=None,
                  device="cuda", chunks: int = 4, graph: bool = True, h2d_streams: int = 1):
        """All ``nranks`` partials on one GPU (the N=1 bench workload)."""
        import torch

        out_dtype = out_dtype or torch.bfloat16

        def make(c):
            op = SimulatedAllReduce(scheme, c, nranks, algo, out_dtype, device)
            return lambda ins, out: op(ins, out)

        return cls(make, n, nranks, torch.bfloat16, out_dtype, device, chunks, graph, h2d_streams)

    @classmethod
    def compressed(cls, scheme, n: int, group=None, algo: str = "oneshot", out_dtype=None,
                   device=None, chunks: int = 4, graph: bool = True, h2d_streams: int = 1):
        """This rank's partial, NCCL exchange (one rank per GPU)."""
        import torch

        out_dtype = out_dtype or torch.bfloat16

        import torch.distributed as dist

        def make(c):
            op = CompressedAllReduce(scheme, c, group=group, algo=algo, out_dtype=out_dtype,
                                     device=device)
            return lambda ins, out: op(ins[0], out)

        pipe = cls(make, n, 1, torch.bfloat16, out_dtype, device or "cuda", chunks, graph,
                   h2d_streams, collective=True)
        if graph and dist.is_initialized() and dist.get_world_size(group) > 1:
            # the communicator exists before the first capture (NCCL cannot
            # be initialised inside a graph capture)
            t = torch.zeros(1, device=pipe.device)
            dist.all_reduce(t, group=group)
            torch.cuda.synchronize(pipe.device)
        return pipe


def simulate_allreduce(partials, scheme, algo: str = "oneshot", out_dtype=None, backend=None):
    """One-off :class:`SimulatedAllReduce`; returns (reduced tensor, nonfinite flag)."""
    sim = SimulatedAllReduce(scheme, partials[0].numel(), len(partials), algo, out_dtype,
                             partials[0].device, backend)
    out = sim(partials)
    return out, sim.flag


# ---------------------------------------------------------------------------
# the reference's wire duck type and analytic model (mx/netbench.py)
# ---------------------------------------------------------------------------


class BlockWire:
    """``_BlockWire`` (mx/netbench.py:146-162) on the GPU codec: same
    ``name`` / ``payload_nbytes`` / ``encode_with_reconstruction`` / ``decode``."""

    def __init__(self, scheme: SchemeDescriptor, shape):
        self.scheme = scheme
        self.shape = tuple(shape)
        self.name = scheme.name

    def payload_nbytes(self) -> int:
        from .codec import serialized_nbytes

        return serialized_nbytes(self.scheme, self.shape)

    def encode_with_reconstruction(self, arr):
        import numpy as np

        from .codec import compress_tensor_device, decompress_tensor_device, serialize

        dct = compress_tensor_device(arr, self.scheme)
        import torch

        own = decompress_tensor_device(dct, torch.float32).cpu().numpy()
        return serialize(dct), own.astype(np.float32, copy=False)

    def decode(self, data: bytes):
        import torch

        from .codec import decompress_tensor_device, deserialize

        return decompress_tensor_device(deserialize(data), torch.float32).cpu().numpy()


# LinkModel / predict_comm_time live in netbench.py (the reference module's
# name); re-exported here for callers of round 1's location
from .netbench import LinkModel, predict_comm_time  # noqa: E402,F401
