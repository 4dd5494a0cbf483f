"""Row-parallel linear hook + TP Llama prefill harness.

Two halves:

1. The reference's simulated reduction (mx/tpsim.py:146-324) -- same names
   and report fields -- with the codec on the GPU:
   ``TPConfig``, ``ReductionReport``, ``shard_rowwise``, ``generate_inputs``,
   ``simulate_reduction``, ``parallelism_sweep``.  Partials are fp32
   ``X[..., rows_r] @ W_r`` (mx/tpsim.py:263), every rank's partial goes
   through the codec (``quantize_own``, 155/268), sums are float64 in rank
   order (275-281) and the triangle-inequality bound is asserted (284-288).

2. The deployment form of the same hook: ``RowParallelLinear`` (o_proj /
   down_proj) whose partial sum is reduced by :class:`CompressedAllReduce`
   (or NCCL bf16 all-reduce when ``scheme`` is None), inside a random-init
   Llama prefill stack (``LlamaTP``) used to measure TTFT.  The GEMMs and
   attention are ordinary cuBLAS / SDPA calls -- not the optimisation target
   (BASELINE.json north_star).
"""

from __future__ import annotations

import os

from dataclasses import dataclass

import numpy as np

from .errors import MinimumDegreeTwo, ShapeMismatch
from .formats import SchemeDescriptor, parse_scheme

UNCOMPRESSED_VALUE_BYTES = 2  # 16-bit activations are the uncompressed baseline


# ---------------------------------------------------------------------------
# 1. simulated reduction (mx/tpsim.py)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class TPConfig:
    """mx/tpsim.py:146-166"""

    degree: int
    scheme: object
    seed: int = 0
    input_shape: tuple = (1, 64, 1024)
    weight_shape: tuple = (1024, 1024)
    quantize_own: bool = True

    def __post_init__(self):
        if self.degree < 2:
            raise MinimumDegreeTwo(f"degree {self.degree} < 2")
        if len(self.input_shape) != 3 or len(self.weight_shape) != 2:
            raise ShapeMismatch("expected (batch, tokens, d_in) and (d_in, d_out)")
        if self.input_shape[2] != self.weight_shape[0]:
            raise ShapeMismatch(f"d_in mismatch: input {self.input_shape[2]}, "
                                f"weight {self.weight_shape[0]}")


@dataclass(frozen=True)
class ReductionReport:
    """mx/tpsim.py:169-190"""

    degree: int
    scheme: str
    rel_frob_err: float
    max_abs_err: float
    sqnr_db: float
    bytes_compressed: int
    bytes_uncompressed: int
    padding: int = 0

    CSV_COLUMNS = ("degree", "scheme", "rel_frob_err", "max_abs_err", "sqnr_db",
                   "bytes_compressed", "bytes_uncompressed")


def shard_rowwise(weight, degree: int):
    """Split (d_in, d_out) into ``degree`` row shards, zero-padding d_in
    (mx/tpsim.py:193-215).  numpy or torch; returns (shards, padding)."""
    if weight.ndim != 2:
        raise ShapeMismatch(f"weight must be 2-D, got shape {tuple(weight.shape)}")
    if degree < 1:
        raise ShapeMismatch("degree must be positive")
    d_in = weight.shape[0]
    rows = -(-d_in // degree)
    pad = rows * degree - d_in
    if pad:
        if isinstance(weight, np.ndarray):
            weight = np.concatenate([weight, np.zeros((pad, weight.shape[1]), weight.dtype)])
        else:
            import torch

            weight = torch.cat([weight, weight.new_zeros(pad, weight.shape[1])])
    return [weight[i * rows:(i + 1) * rows] for i in range(degree)], pad


def generate_inputs(cfg: TPConfig):
    """Seeded activations with outliers and N(0,1) weights (mx/tpsim.py:218-223)."""
    from .synth import gaussian_with_outliers

    rng = np.random.default_rng(cfg.seed)
    x = gaussian_with_outliers(rng, cfg.input_shape)
    w = rng.standard_normal(cfg.weight_shape).astype(np.float32)
    return x, w


def _sqnr_db(ref: np.ndarray, err: np.ndarray) -> float:
    e = float(np.sum(np.square(err)))
    if e == 0.0:
        return float("inf")
    return 10.0 * np.log10(float(np.sum(np.square(ref))) / e)  # as mx/tpsim.py:231


class _MxCodec:
    """MX block codec on the GPU (mx/tpsim.py:51-63)."""

    def __init__(self, scheme: SchemeDescriptor):
        self.scheme = scheme
        self.name = scheme.name

    def encode(self, arr) -> bytes:
        from .codec import compress_tensor, serialize

        return serialize(compress_tensor(np.asarray(arr), self.scheme))

    def decode(self, data: bytes, shape) -> np.ndarray:
        from .codec import decompress_tensor, deserialize

        out = decompress_tensor(deserialize(data))
        if out.shape != tuple(shape):
            raise ShapeMismatch(f"payload shape {out.shape} != expected {tuple(shape)}")
        return out

    def roundtrip(self, p: np.ndarray):
        """(float64 reconstruction, payload bytes) without host byte streams."""
        import torch

        from .codec import (_download, _upload_array, compress_tensor_device,
                            decompress_tensor_device, serialized_nbytes)

        dct = compress_tensor_device(_upload_array(torch.from_numpy(np.ascontiguousarray(p))),
                                     self.scheme)
        rec = _download(decompress_tensor_device(dct, torch.float64))
        return rec, serialized_nbytes(self.scheme, p.shape)


class _PassthroughCodec:
    """Raw float32 bytes (mx/tpsim.py:66-82): numerically the identity."""

    name = "passthrough"

    def encode(self, arr) -> bytes:
        from .codec import FORMAT_CODE_RAW_F32, pack_header

        a = np.asarray(arr)
        return pack_header(FORMAT_CODE_RAW_F32, 0, 0, tuple(a.shape)) + \
            np.ascontiguousarray(a, dtype="<f4").tobytes()

    def decode(self, data: bytes, shape) -> np.ndarray:
        from .codec import unpack_header

        _, _, _, wshape, off = unpack_header(data)
        n = int(np.prod(wshape, dtype=np.int64))
        return np.frombuffer(data, "<f4", count=n, offset=off).astype(np.float64).reshape(wshape)

    def roundtrip(self, p: np.ndarray):
        from .codec import header_nbytes

        return p.astype(np.float32).astype(np.float64), header_nbytes(p.ndim) + 4 * p.size


class _Fp16Codec:
    """IEEE half round trip (mx/tpsim.py:85-100), the 16-bit wire baseline;
    the cast runs on the GPU."""

    name = "fp16"

    def encode(self, arr) -> bytes:
        from .codec import FORMAT_CODE_RAW_F16, pack_header

        a = np.asarray(arr)
        h = self._half(a)
        return pack_header(FORMAT_CODE_RAW_F16, 0, 0, tuple(a.shape)) + h.astype("<f2").tobytes()

    def decode(self, data: bytes, shape) -> np.ndarray:
        from .codec import unpack_header

        _, _, _, wshape, off = unpack_header(data)
        n = int(np.prod(wshape, dtype=np.int64))
        return np.frombuffer(data, "<f2", count=n, offset=off).astype(np.float64).reshape(wshape)

    @staticmethod
    def _half(a: np.ndarray) -> np.ndarray:
        import torch

        from . import _native

        _native.require_cuda()
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()
        return t.to(torch.float16).cpu().numpy()  # one RNE rounding from float64

    def roundtrip(self, p: np.ndarray):
        from .codec import header_nbytes

        return self._half(p).astype(np.float64), header_nbytes(p.ndim) + 2 * p.size


class _TopKCodec:
    """TopK on the GPU (mx/tpsim.py:100-109)."""

    def __init__(self, factor: float):
        self.factor = factor
        self.name = f"topk:{factor:g}"

    def encode(self, arr) -> bytes:
        from . import baselines as bl

        return bl.serialize_topk(bl.topk_compress(arr, self.factor))

    def decode(self, data: bytes, shape) -> np.ndarray:
        from . import baselines as bl

        return bl.topk_decompress(bl.deserialize_topk(data))

    def roundtrip(self, p: np.ndarray):
        import torch

        from . import baselines as bl
        from .codec import _download, header_nbytes

        k = bl.topk_budget(p.size, p.ndim, self.factor)
        if self.factor <= 1 or k < 1:
            from .errors import CompressionFactorTooHigh

            raise CompressionFactorTooHigh(f"factor {self.factor} leaves room for {k} values")
        idx, val = bl.topk_compress_device(torch.from_numpy(np.ascontiguousarray(p)), k)
        rec = _download(bl.topk_decompress_device(idx, val, p.size, torch.float64))
        return rec.reshape(p.shape), header_nbytes(p.ndim) + 6 * idx.numel()


class _ChannelIntCodec:
    """Channel-wise INT on the GPU (mx/tpsim.py:112-125)."""

    def __init__(self, bits: int):
        self.bits = bits
        self.name = f"chanint:{bits}"

    def encode(self, arr) -> bytes:
        from . import baselines as bl

        return bl.serialize_channel_int(bl.channelwise_int_compress(arr, self.bits))

    def decode(self, data: bytes, shape) -> np.ndarray:
        from . import baselines as bl

        return bl.channelwise_int_decompress(bl.deserialize_channel_int(data))

    def roundtrip(self, p: np.ndarray):
        import torch

        from . import baselines as bl
        from .codec import _download, header_nbytes

        s, c, shape = bl.channelwise_int_compress_device(torch.from_numpy(np.ascontiguousarray(p)),
                                                         self.bits)
        rec = bl.channelwise_int_decompress_device(s, c, shape, self.bits, torch.float64)
        return (_download(rec).reshape(p.shape),
                header_nbytes(p.ndim) + 2 * s.numel() + c.numel())


def resolve_codec(scheme, extensions: bool = False):
    """A SchemeDescriptor or codec id -> codec object (mx/tpsim.py:128-143):
    MX schemes, ``passthrough``/``none``, ``fp16``, ``topk:F``, ``chanint:B``.
    Scheme ids resolve through the reference registry, so unknown ids (and
    the FP6 / INT8 extension formats) raise UnknownScheme as in the
    reference; ``extensions=True`` opts in to the extension formats."""
    from .errors import UnknownScheme

    if isinstance(scheme, SchemeDescriptor):
        return _MxCodec(scheme)
    if not isinstance(scheme, str):
        raise UnknownScheme(f"cannot interpret {scheme!r} as a codec")
    name = scheme.strip().lower()
    if name in ("passthrough", "none"):
        return _PassthroughCodec()
    if name == "fp16":
        return _Fp16Codec()
    if name.startswith("topk:"):
        return _TopKCodec(float(name.split(":", 1)[1]))
    if name.startswith("chanint:"):
        return _ChannelIntCodec(int(name.split(":", 1)[1]))
    return _MxCodec(parse_scheme(name, extensions=extensions))


def simulate_reduction(cfg: TPConfig, x=None, w=None, partials_on_gpu: bool = False,
                       partials=None):
    """One compress/exchange/decompress/reduce cycle, scored (mx/tpsim.py:234-302).

    The codec (any id of :func:`resolve_codec`) runs on the GPU.  Partials
    are computed with numpy (bit-identical to the reference) unless
    ``partials_on_gpu`` (cuBLAS fp32, faster, sums differ in the last bits).
    ``partials`` injects precomputed fp32 partial products (one per rank) --
    BLAS results depend on the host CPU, so parity tests replay the
    reference's own partials."""
    import torch

    if x is None or w is None:
        gx, gw = generate_inputs(cfg)
        x = gx if x is None else x
        w = gw if w is None else w
    x = np.asarray(x, dtype=np.float32)
    w = np.asarray(w, dtype=np.float32)
    if x.shape[-1] != w.shape[0]:
        raise ShapeMismatch(f"d_in mismatch: {x.shape[-1]} vs {w.shape[0]}")
    shards, padding = shard_rowwise(w, cfg.degree)
    if padding:
        x = np.pad(x, [(0, 0)] * (x.ndim - 1) + [(0, padding)])
    rows = shards[0].shape[0]
    wire = resolve_codec(cfg.scheme)
    given = partials
    partials, decoded = [], []
    payload = None
    for r in range(cfg.degree):
        xs = x[..., r * rows:(r + 1) * rows]
        if given is not None:
            p = np.asarray(given[r], dtype=np.float32)
        elif partials_on_gpu:
            p = (torch.from_numpy(np.ascontiguousarray(xs)).cuda()
                 @ torch.from_numpy(shards[r]).cuda()).cpu().numpy()
        else:
            p = xs @ shards[r]  # float32, like the deployed matmul (tpsim.py:263)
        partials.append(p)
        rec, nbytes = wire.roundtrip(p)
        if payload is None:
            payload = nbytes
        decoded.append(rec if (cfg.quantize_own or r != 0) else p.astype(np.float64))
    ref = np.zeros(partials[0].shape, np.float64)
    red = np.zeros_like(ref)
    per = np.zeros_like(ref)
    for r in range(cfg.degree):  # float64, rank order (tpsim.py:275-281)
        ref += partials[r].astype(np.float64)
        red += decoded[r]
        per += np.abs(decoded[r] - partials[r].astype(np.float64))
    err = red - ref
    tol = 1e-9 * (np.abs(ref) + 1.0)
    if not (np.abs(err) <= per + tol).all():  # tpsim.py:284-288
        raise AssertionError("summed error exceeded per-worker error budget")
    en, rn = float(np.linalg.norm(err.ravel())), float(np.linalg.norm(ref.ravel()))
    return ReductionReport(
        degree=cfg.degree, scheme=wire.name, rel_frob_err=0.0 if en == 0.0 else en / rn,
        max_abs_err=float(np.max(np.abs(err))), sqnr_db=_sqnr_db(ref, err),
        bytes_compressed=(cfg.degree - 1) * int(payload),
        bytes_uncompressed=(cfg.degree - 1) * ref.size * UNCOMPRESSED_VALUE_BYTES,
        padding=padding)


def parallelism_sweep(cfg: TPConfig, degrees):
    """mx/tpsim.py:305-324"""
    degrees = list(degrees)
    if not degrees:
        raise MinimumDegreeTwo("no degrees requested")
    for d in degrees:
        if d < 2:
            raise MinimumDegreeTwo(f"degree {d} < 2")
    return [simulate_reduction(TPConfig(d, cfg.scheme, cfg.seed, cfg.input_shape,
                                        cfg.weight_shape, cfg.quantize_own)) for d in degrees]


# ---------------------------------------------------------------------------
# 2. TP Llama prefill with the compressed row-parallel hook
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class LlamaConfig:
    hidden: int
    ffn: int
    layers: int
    heads: int
    kv_heads: int
    vocab: int = 128256
    rope_theta: float = 500000.0
    eps: float = 1e-5

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads


LLAMA31_8B = LlamaConfig(4096, 14336, 32, 32, 8)
LLAMA31_70B = LlamaConfig(8192, 28672, 80, 64, 8)


def _torch():
    import torch

    return torch


_SYMM_CACHE = {}  # (group, scheme, n, dtype, algo) -> SymmetricAllReduce shared by layers
_PUSH_CACHE = {}  # (group, scheme, n, dtype) -> FusedLinearAllReduce shared by layers


def make_module_classes():
    """Build the nn.Module classes lazily (torch import stays optional for
    the pure-host parts of the package)."""
    torch = _torch()
    nn = torch.nn
    F = torch.nn.functional

    class RowParallelLinear(nn.Module):
        """y = all_reduce(x_local @ W_r): the hook of mx/tpsim.py:263-281.

        ``scheme`` None -> uncompressed NCCL bf16 all-reduce; otherwise the
        MX-compressed all-reduce: ``algo`` "oneshot" / "twoshot" over NCCL,
        "symm" / "symm2" for the one-kernel NVLink forms (K5 / K5b, one
        symmetric buffer shared by every layer of the same shape), "auto"
        for one-shot up to TP=2 and two-shot beyond."""

        def __init__(self, d_in_local, d_out, group=None, scheme=None, algo="oneshot",
                     tokens=None, device="cuda", dtype=torch.bfloat16, std=0.02,
                     fused_gemm=None, shared_collectives=None):
            super().__init__()
            self.weight = nn.Parameter(torch.randn(d_out, d_in_local, device=device, dtype=dtype)
                                       * std, requires_grad=False)
            self.group, self.scheme, self.algo = group, scheme, algo
            # the quantiser fused into the GEMM epilogue (k_gemm.cu) for the
            # NCCL algorithms: "auto" where it is expected to win
            # (NativeBackend.gemm_preferred), True always, False never
            # (F.linear + K1); MXB200_GEMM_FUSED=0/1 pins False/True
            env = os.environ.get("MXB200_GEMM_FUSED")
            self.fused_gemm = fused_gemm if fused_gemm is not None else (
                "auto" if env is None else env != "0")
            # the residual add fused into the dequant-sum store;
            # MXB200_FUSE_RESIDUAL=0 adds after the collective instead
            self.fuse_residual = os.environ.get("MXB200_FUSE_RESIDUAL", "1") != "0"
            self._car = {}
            # a dict shared by the layers of one model (LlamaTP): one set of
            # collective buffers per (group, shape, scheme, algo) instead of
            # one per layer -- layers run one after another on the stream,
            # and the residual-fused reduce updates h in place (its output
            # aliasing its residual is allowed).  Without it every layer owns
            # its buffers (the output of one call stays valid until that
            # layer's next call).
            self._shared = shared_collectives

        def _collective(self, n, dtype, device):
            import torch.distributed as dist

            from .collective import CompressedAllReduce, SymmetricAllReduce

            key = (n, dtype, str(self.scheme), self.algo)
            car = self._car.get(key)
            if car is None and self._shared is not None:
                car = self._shared.get((id(self.group),) + key)
            if car is None:
                ws = dist.get_world_size(self.group) if dist.is_initialized() else 1
                rk = dist.get_rank(self.group) if dist.is_initialized() else 0
                algo = self.algo
                if algo == "auto":
                    algo = "oneshot" if ws <= 2 else "twoshot"
                if algo == "push":  # operands the push GEMM cannot take: K5
                    algo = "symm"
                if algo in ("symm", "symm2"):
                    skey = (id(self.group), str(self.scheme), n, dtype, algo)
                    car = _SYMM_CACHE.get(skey)
                    if car is None:
                        car = SymmetricAllReduce(self.scheme, n, group=self.group,
                                                 out_dtype=dtype, device=device,
                                                 algo="oneshot" if algo == "symm" else "twoshot")
                        _SYMM_CACHE[skey] = car
                else:
                    car = CompressedAllReduce(self.scheme, n, group=self.group,
                                              algo=algo, out_dtype=dtype, device=device,
                                              world_size=ws, rank=rk)
                if self._shared is not None:
                    self._shared[(id(self.group),) + key] = car
                self._car[key] = car
            return car

        def reduce(self, y, residual=None):
            import torch.distributed as dist

            if self.scheme is None:
                if dist.is_initialized() and dist.get_world_size(self.group) > 1:
                    dist.all_reduce(y, group=self.group)
                return y if residual is None else residual + y
            car = self._collective(y.numel(), y.dtype, y.device)
            if residual is None or not self.fuse_residual:
                out = car(y.contiguous())
                return out if residual is None else residual + out
            return car(y.contiguous(), residual=residual.contiguous())

        def _push(self, n, dtype, device):
            import torch.distributed as dist

            from .collective import FusedLinearAllReduce

            key = (id(self.group), str(self.scheme), n, dtype)
            fl = _PUSH_CACHE.get(key)
            if fl is None:
                ws = dist.get_world_size(self.group)
                algo = "oneshot" if ws <= 2 or n % (1024 * ws) else "twoshot"
                fl = FusedLinearAllReduce(self.scheme, n, group=self.group, out_dtype=dtype,
                                          device=device, algo=algo)
                _PUSH_CACHE[key] = fl
            self._car[("push",) + key] = fl
            return fl

        def forward(self, x, residual=None):
            """all_reduce(x @ W^T), or ``residual + all_reduce(x @ W^T)`` --
            the Llama block's residual update -- with the add fused into the
            compressed collective's dequant-sum store (the bf16 NCCL path
            adds after the all-reduce; identical bits either way).
            ``algo="push"``: the GEMM, the quantiser and the all-gather
            (one-shot to TP=2) or the reduce-scatter leg (two-shot beyond)
            in one kernel (FusedLinearAllReduce), K5 where it does not apply."""
            if self.scheme is not None and self.algo == "push":
                n = x.numel() // x.shape[-1] * self.weight.shape[0]
                fl = self._push(n, x.dtype, x.device)
                xc = x.contiguous()
                if fl.supported(xc, self.weight):
                    if residual is not None and not self.fuse_residual:
                        return residual + fl.linear(xc, self.weight)
                    return fl.linear(xc, self.weight,
                                     residual=None if residual is None else residual.contiguous())
            if self.scheme is not None and self.fused_gemm and self.algo not in ("symm", "symm2",
                                                                                  "push"):
                n = x.numel() // x.shape[-1] * self.weight.shape[0]
                car = self._collective(n, x.dtype, x.device)
                if hasattr(car, "linear") and (
                        self.fused_gemm != "auto" or
                        car.backend.gemm_preferred(x.reshape(-1, x.shape[-1]), self.weight)):
                    if residual is None or not self.fuse_residual:
                        out = car.linear(x.contiguous(), self.weight)
                        return out if residual is None else residual + out
                    return car.linear(x.contiguous(), self.weight,
                                      residual=residual.contiguous())
            return self.reduce(F.linear(x, self.weight), residual)

        def collectives(self):
            return list(self._car.values())

    def check_collectives(cars):
        """Deferred health check of compressed all-reduces: ONE device->host
        read covers every op's sticky non-finite flag and every NVLink op's
        peer-wait status; raises NonFiniteInput / RuntimeError (a timed-out
        peer wait means that call's result is invalid)."""
        cars = list({id(c): c for c in cars}.values())
        if not cars:
            return
        parts = [c.flag.reshape(1) for c in cars]
        symm = [c for c in cars if hasattr(c, "state")]
        parts += [c.state[:1].to(torch.int64) for c in symm]
        v = torch.cat(parts).cpu().tolist()
        for c, s in zip(symm, v[len(cars):]):
            if s != 0:
                c.check_status()
        for c, f in zip(cars, v[:len(cars)]):
            if f >= 0:
                c.check_finite()

    class ColumnParallelLinear(nn.Module):
        def __init__(self, d_in, d_out_local, device="cuda", dtype=torch.bfloat16, std=0.02):
            super().__init__()
            self.weight = nn.Parameter(torch.randn(d_out_local, d_in, device=device, dtype=dtype)
                                       * std, requires_grad=False)

        def forward(self, x):
            return F.linear(x, self.weight)

    class RMSNorm(nn.Module):
        def __init__(self, d, eps, device, dtype):
            super().__init__()
            self.w = nn.Parameter(torch.ones(d, device=device, dtype=dtype), requires_grad=False)
            self.eps = eps

        def forward(self, x):
            xf = x.float()
            return (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + self.eps)).to(x.dtype) \
                * self.w

    class LlamaTPBlock(nn.Module):
        def __init__(self, cfg: LlamaConfig, tp: int, group, scheme, algo, device, dtype,
                     fused_gemm=None, shared_collectives=None):
            super().__init__()
            if cfg.heads % tp or cfg.kv_heads % tp and tp % cfg.kv_heads:
                raise ShapeMismatch(f"heads {cfg.heads}/{cfg.kv_heads} vs tp {tp}")
            self.hl = cfg.heads // tp
            self.kvl = max(1, cfg.kv_heads // tp)
            self.hd = cfg.head_dim
            self.cfg = cfg
            self.ln1 = RMSNorm(cfg.hidden, cfg.eps, device, dtype)
            self.ln2 = RMSNorm(cfg.hidden, cfg.eps, device, dtype)
            self.qkv = ColumnParallelLinear(cfg.hidden, (self.hl + 2 * self.kvl) * self.hd,
                                            device, dtype)
            self.o_proj = RowParallelLinear(self.hl * self.hd, cfg.hidden, group, scheme, algo,
                                            device=device, dtype=dtype, fused_gemm=fused_gemm,
                                            shared_collectives=shared_collectives)
            self.gate_up = ColumnParallelLinear(cfg.hidden, 2 * (cfg.ffn // tp), device, dtype)
            self.down_proj = RowParallelLinear(cfg.ffn // tp, cfg.hidden, group, scheme, algo,
                                               device=device, dtype=dtype, fused_gemm=fused_gemm,
                                               shared_collectives=shared_collectives)

        def forward(self, h, cos, sin):
            b, t, _ = h.shape
            x = self.ln1(h)
            qkv = self.qkv(x).view(b, t, self.hl + 2 * self.kvl, self.hd)
            q, k, v = qkv.split([self.hl, self.kvl, self.kvl], dim=2)
            q, k = _rope(q, cos, sin), _rope(k, cos, sin)
            q, k, v = (z.transpose(1, 2) for z in (q, k, v))
            a = F.scaled_dot_product_attention(q, k, v, is_causal=True,
                                               enable_gqa=self.hl != self.kvl)
            h = self.o_proj(a.transpose(1, 2).reshape(b, t, self.hl * self.hd), residual=h)
            g, u = self.gate_up(self.ln2(h)).chunk(2, dim=-1)
            return self.down_proj(F.silu(g) * u, residual=h)

    def _rope(x, cos, sin):
        x1, x2 = x[..., : x.shape[-1] // 2], x[..., x.shape[-1] // 2:]
        return (x * cos + torch.cat([-x2, x1], dim=-1) * sin).to(x.dtype)

    class LlamaTP(nn.Module):
        """Random-init Llama prefill stack, TP-sharded (no embedding/LM head:
        TTFT of the transformer body, where the all-reduces live)."""

        def __init__(self, cfg: LlamaConfig, tp: int = 1, group=None, scheme=None,
                     algo="oneshot", layers=None, device="cuda", dtype=torch.bfloat16,
                     check_health: bool = True, fused_gemm=None):
            super().__init__()
            self.cfg = cfg
            self.check_health = check_health
            self._shared_collectives = {}  # one buffer set per shape/scheme for all layers
            self.blocks = nn.ModuleList(LlamaTPBlock(cfg, tp, group, scheme, algo, device, dtype,
                                                     fused_gemm, self._shared_collectives)
                                        for _ in range(layers or cfg.layers))
            self.norm = RMSNorm(cfg.hidden, cfg.eps, device, dtype)

        def rope_cache(self, t, device, dtype):
            hd = self.cfg.head_dim
            inv = 1.0 / (self.cfg.rope_theta ** (torch.arange(0, hd, 2, device=device).float()
                                                 / hd))
            ang = torch.outer(torch.arange(t, device=device).float(), inv)
            ang = torch.cat([ang, ang], dim=-1)[None, :, None, :]
            return ang.cos().to(dtype), ang.sin().to(dtype)

        def forward(self, h):
            cos, sin = self.rope_cache(h.shape[1], h.device, h.dtype)
            for blk in self.blocks:
                h = blk(h, cos, sin)
            out = self.norm(h)
            # once per forward: the compressed all-reduces' sticky non-finite
            # flags and NVLink peer-wait status (one host read; skipped while
            # a CUDA graph is being captured -- check_collectives() after
            # the replays instead)
            if self.check_health and not torch.cuda.is_current_stream_capturing():
                self.check_collectives()
            return out

        def configure(self, scheme, algo="oneshot", fused_gemm=None):
            """Switch every row-parallel layer to another all-reduce (bf16 NCCL
            when ``scheme`` is None) on the SAME weights; collectives are
            cached per (shape, scheme, algo), so switching back reuses them."""
            for blk in self.blocks:
                for m in (blk.o_proj, blk.down_proj):
                    m.scheme, m.algo = scheme, algo
                    if fused_gemm is not None:
                        m.fused_gemm = fused_gemm
            return self

        def collectives(self):
            return [c for blk in self.blocks for m in (blk.o_proj, blk.down_proj)
                    for c in m.collectives()]

        def check_collectives(self):
            check_collectives(self.collectives())

    return RowParallelLinear, ColumnParallelLinear, LlamaTPBlock, LlamaTP


def measure_ttft(cfg: LlamaConfig, batch: int, seq: int, tp: int = 1, group=None, scheme=None,
                 algo="oneshot", layers=None, reps: int = 5, warmup: int = 2, seed: int = 0,
                 graph: bool = False, fused_gemm=None):
    """Prefill latency (ms, max over ranks) of the TP body on random data.
    ``graph`` replays the whole forward as one captured CUDA graph (how a
    serving engine runs it: no per-kernel host launch cost)."""
    torch = _torch()
    import torch.distributed as dist

    torch.manual_seed(seed)
    _, _, _, LlamaTP = make_module_classes()
    model = LlamaTP(cfg, tp, group, scheme, algo, layers, fused_gemm=fused_gemm)
    h = torch.randn(batch, seq, cfg.hidden, device="cuda", dtype=torch.bfloat16)
    with torch.inference_mode():
        for _ in range(warmup):
            model(h)
        torch.cuda.synchronize()
        run = lambda: model(h)  # noqa: E731
        if graph:
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                model(h)
            torch.cuda.current_stream().wait_stream(s)
            torch.cuda.synchronize()
            with torch.cuda.graph(g):
                model(h)
            run = g.replay
        if dist.is_initialized():
            dist.barrier(group)
        times = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run()
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        # graph replays skip the per-forward check: one check after them
        model.check_collectives()
    ms = float(np.median(times))
    if dist.is_initialized():
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        ms = float(t.item())
    return ms


def measure_ttft_ab(cfg: LlamaConfig, batch: int, seq: int, variants, tp: int = 1, group=None,
                    layers=None, reps: int = 15, warmup: int = 2, seed: int = 0):
    """Prefill TTFT of several all-reduce variants on ONE model (same
    weights, same input), each captured as its own CUDA graph, the replays
    interleaved round-robin (v0 v1 v2 v0 v1 v2 ...) so clock / thermal drift
    hits every variant alike.  ``variants``: [(label, scheme | None, algo,
    fused_gemm)].  Returns {label: median ms (max over ranks)}; a variant
    that fails to build or capture maps to the exception text."""
    torch = _torch()
    import torch.distributed as dist

    torch.manual_seed(seed)
    _, _, _, LlamaTP = make_module_classes()
    model = LlamaTP(cfg, tp, group, None, "oneshot", layers)
    h = torch.randn(batch, seq, cfg.hidden, device="cuda", dtype=torch.bfloat16)
    graphs, errors = {}, {}
    with torch.inference_mode():
        for label, scheme, algo, fused in variants:
            try:
                model.configure(scheme, algo, fused)
                for _ in range(warmup):
                    model(h)
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                s = torch.cuda.Stream()
                s.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(s):
                    model(h)
                torch.cuda.current_stream().wait_stream(s)
                torch.cuda.synchronize()
                with torch.cuda.graph(g):
                    model(h)
                graphs[label] = g
            except Exception as exc:  # noqa: BLE001 (reported per variant)
                errors[label] = f"{type(exc).__name__}: {exc}"[:200]
                torch.cuda.synchronize()
        if dist.is_initialized():
            # every rank must run the same graphs in the same order
            ok = torch.tensor([len(graphs)], device="cuda")
            dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
            if int(ok.item()) != len(graphs):
                raise RuntimeError(f"variants failed on another rank: {errors}")
            dist.barrier(group)
        times = {label: [] for label in graphs}
        for label, g in graphs.items():
            g.replay()
        torch.cuda.synchronize()
        for _ in range(reps):
            for label, g in graphs.items():
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                times[label].append(e0.elapsed_time(e1))
        model.check_collectives()
    out = {}
    for label in graphs:
        ms = float(np.median(times[label]))
        if dist.is_initialized():
            t = torch.tensor([ms], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
            ms = float(t.item())
        out[label] = ms
    out.update(errors)
    del graphs
    return out
