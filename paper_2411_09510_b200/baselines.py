"""Comparison codecs -- TopK sparsification and channel-wise INT -- on the
sm_100a kernels (k_baselines.cu), with the reference's API (mx/baselines.py).

Same names, argument meaning, return types and errors as the reference:
``topk_budget``, ``topk_compress`` / ``topk_decompress``,
``channelwise_int_compress`` / ``channelwise_int_decompress``, the packets
and their MXC1 containers (format codes 0xF0 / 0xF1).  Packets hold host
arrays / bytes like the reference's; the ``*_device`` variants keep
everything on the GPU (the form a compressed collective would use).
These are the paper's Table 4 baselines.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .codec import (FORMAT_CODE_CHANNEL_INT, FORMAT_CODE_TOPK, _download, _dtype_code, _stream,
                    _to_device_values, _upload_array, header_nbytes, pack_header, packed_nbytes,
                    unpack_header)
from .errors import CompressionFactorTooHigh, MalformedHeader, NonFiniteInput, TruncatedStream

TOPK_INDEX_BYTES = 4
TOPK_VALUE_BYTES = 2
ORIGINAL_VALUE_BYTES = 2  # baselines compete against 16-bit uncompressed tensors


@dataclass(frozen=True)
class TopKPacket:
    """mx/baselines.py:38-60"""

    shape: tuple
    indices: np.ndarray  # uint32, ascending
    values: np.ndarray  # float16

    def __post_init__(self):
        if self.indices.shape != self.values.shape:
            raise ValueError("indices and values must pair up one to one")

    @property
    def k_per_tensor(self) -> int:
        return int(self.indices.size)

    @property
    def nbytes(self) -> int:
        return header_nbytes(len(self.shape)) + self.k_per_tensor * (
            TOPK_INDEX_BYTES + TOPK_VALUE_BYTES)


@dataclass(frozen=True)
class ChannelIntPacket:
    """mx/baselines.py:63-78"""

    shape: tuple
    bits: int
    scales: np.ndarray  # float16 per trailing-dimension channel
    code_stream: bytes

    @property
    def nbytes(self) -> int:
        return header_nbytes(len(self.shape)) + 2 * self.scales.size + len(self.code_stream)


def _torch():
    import torch

    return torch


def _p(t):
    return ctypes.c_void_p(t.data_ptr())


def _nonfinite_flag():
    torch = _torch()
    flag = torch.empty(1, dtype=torch.int64, device="cuda")
    _native.check(_native.load().mx_nonfinite_reset(_p(flag), _stream()), "mx_nonfinite_reset")
    return flag


def _check_flag(flag):
    idx = int(flag.item())
    if idx >= 0:  # UINT64_MAX reads as -1: no NaN/Inf seen
        raise NonFiniteInput(f"non-finite value at flat index {idx}")


# ---------------------------------------------------------------------------
# TopK (mx/baselines.py:88-135)
# ---------------------------------------------------------------------------


def topk_budget(total_elements: int, ndim: int, compression_factor: float) -> int:
    """Largest K whose packet fits original_bytes / factor (mx/baselines.py:88-92)."""
    original = total_elements * ORIGINAL_VALUE_BYTES
    budget = original / compression_factor - header_nbytes(ndim)
    return int(budget // (TOPK_INDEX_BYTES + TOPK_VALUE_BYTES))


def topk_compress_device(x, k: int, check_finite: bool = True):
    """Device TopK of a CUDA/host tensor: (indices u32 as int32 tensor,
    f16 values tensor), K entries in ascending index order."""
    torch = _torch()
    lib = _native.load()
    xd, _ = _to_device_values(x)
    n = xd.numel()
    k = int(min(k, n))
    idx = torch.empty(k, dtype=torch.int32, device="cuda")
    val = torch.empty(k, dtype=torch.float16, device="cuda")
    if k == 0:
        return idx, val
    wsb = ctypes.c_int64()
    _native.check(lib.mx_topk_workspace_bytes(n, ctypes.byref(wsb)), "mx_topk_workspace_bytes")
    ws = torch.empty(wsb.value, dtype=torch.uint8, device="cuda")
    flag = _nonfinite_flag() if check_finite else None
    _native.check(lib.mx_topk_compress(_p(xd), _dtype_code(xd), n, k, _p(idx), _p(val), _p(ws),
                                       wsb.value, _p(flag) if flag is not None else None,
                                       _stream()), "mx_topk_compress")
    if check_finite:
        _check_flag(flag)
    return idx, val


def topk_compress(tensor, compression_factor: float | None = None, *,
                  k: int | None = None) -> TopKPacket:
    """Keep the K largest magnitudes, ties toward the lower index
    (mx/baselines.py:95-128), selected on the GPU."""
    arr_shape = tuple(int(d) for d in np.shape(tensor))
    n = int(np.prod(arr_shape, dtype=np.int64)) if arr_shape else 1
    if k is None:
        if compression_factor is None:
            raise ValueError("pass compression_factor or k")
        if compression_factor <= 1:
            raise CompressionFactorTooHigh(
                f"compression factor must exceed 1, got {compression_factor}")
        k = topk_budget(n, len(arr_shape), compression_factor)
    if k < 1:
        raise CompressionFactorTooHigh(f"factor {compression_factor} leaves room for {k} values")
    k = min(k, n)
    idx, val = topk_compress_device(tensor, k)
    return TopKPacket(shape=arr_shape, indices=_download(idx).view(np.uint32).copy(),
                      values=_download(val).copy())


def topk_decompress_device(indices, values, n: int, dtype=None):
    torch = _torch()
    dtype = dtype or torch.float64
    out = torch.empty(n, dtype=dtype, device="cuda")
    idx = _upload_array(torch.as_tensor(indices).contiguous())
    val = _upload_array(torch.as_tensor(values).contiguous())
    if idx.dtype != torch.int32:
        idx = idx.to(torch.int64).to(torch.int32)
    val = val.view(torch.float16) if val.dtype == torch.float16 else val.to(torch.float16)
    _native.check(_native.load().mx_topk_decompress(
        _p(idx), _p(val), idx.numel(), n, _p(out), _dtype_code(out), _stream()),
        "mx_topk_decompress")
    return out


def topk_decompress(packet: TopKPacket) -> np.ndarray:
    """Scatter the kept f16 values into zeros (mx/baselines.py:131-135)."""
    torch = _torch()
    n = int(np.prod(packet.shape, dtype=np.int64)) if packet.shape else 1
    idx = torch.from_numpy(np.ascontiguousarray(packet.indices, dtype=np.uint32).view(np.int32))
    val = torch.from_numpy(np.ascontiguousarray(packet.values, dtype=np.float16))
    out = topk_decompress_device(idx, val, n, torch.float64)
    return _download(out).reshape(packet.shape)


def serialize_topk(packet: TopKPacket) -> bytes:
    header = pack_header(FORMAT_CODE_TOPK, 0, packet.k_per_tensor, packet.shape)
    return header + packet.indices.astype("<u4").tobytes() + packet.values.astype("<f2").tobytes()


def deserialize_topk(data: bytes) -> TopKPacket:
    format_code, _, k, shape, offset = unpack_header(data)
    if format_code != FORMAT_CODE_TOPK:
        raise MalformedHeader(f"format code {format_code:#x} is not TopK")
    idx_end = offset + k * TOPK_INDEX_BYTES
    val_end = idx_end + k * TOPK_VALUE_BYTES
    if len(data) < val_end:
        raise TruncatedStream(f"TopK payload needs {val_end} bytes, got {len(data)}")
    return TopKPacket(shape=shape,
                      indices=np.frombuffer(data, "<u4", count=k, offset=offset).copy(),
                      values=np.frombuffer(data, "<f2", count=k, offset=idx_end).copy())


# ---------------------------------------------------------------------------
# channel-wise INT (mx/baselines.py:138-178)
# ---------------------------------------------------------------------------


def channelwise_int_compress_device(x, bits: int = 4, check_finite: bool = True):
    """(f16 scales tensor [C], packed code tensor uint8, shape) on the GPU."""
    torch = _torch()
    if not 2 <= bits <= 8:
        raise ValueError(f"bits must be in [2, 8], got {bits}")
    xd, shape = _to_device_values(x)
    if len(shape) == 0:
        shape = (1,)
    C = shape[-1]
    rows = xd.numel() // C if C else 0
    scales = torch.empty(C, dtype=torch.float16, device="cuda")
    codes = torch.empty(packed_nbytes(xd.numel(), bits), dtype=torch.uint8, device="cuda")
    ws = torch.empty(8 * max(C, 1), dtype=torch.uint8, device="cuda")
    flag = _nonfinite_flag() if check_finite else None
    _native.check(_native.load().mx_chanint_compress(
        _p(xd), _dtype_code(xd), rows, C, bits, _p(scales), _p(codes), _p(ws), ws.numel(),
        _p(flag) if flag is not None else None, _stream()), "mx_chanint_compress")
    if check_finite:
        _check_flag(flag)
    return scales, codes, shape


def channelwise_int_compress(tensor, bits: int = 4) -> ChannelIntPacket:
    """Symmetric per-channel INT along the trailing dimension (mx/baselines.py:138-168)."""
    scales, codes, shape = channelwise_int_compress_device(tensor, bits)
    orig = tuple(int(d) for d in np.shape(tensor))
    return ChannelIntPacket(shape=orig or (1,), bits=bits, scales=_download(scales).copy(),
                            code_stream=_download(codes).tobytes())


def channelwise_int_decompress_device(scales, codes, shape, bits: int, dtype=None):
    torch = _torch()
    dtype = dtype or torch.float64
    n = int(np.prod(shape, dtype=np.int64))
    C = int(shape[-1])
    out = torch.empty(n, dtype=dtype, device="cuda")
    s = _upload_array(torch.as_tensor(scales).contiguous())
    s = s if s.dtype == torch.float16 else s.to(torch.float16)
    c = _upload_array(torch.as_tensor(codes).contiguous())
    _native.check(_native.load().mx_chanint_decompress(
        _p(s), _p(c), n // C if C else 0, C, bits, _p(out), _dtype_code(out), _stream()),
        "mx_chanint_decompress")
    return out.reshape(shape)


def channelwise_int_decompress(packet: ChannelIntPacket) -> np.ndarray:
    """level * scale in float64 (mx/baselines.py:171-178)."""
    torch = _torch()
    codes = torch.from_numpy(np.frombuffer(packet.code_stream, dtype=np.uint8).copy())
    scales = torch.from_numpy(np.ascontiguousarray(packet.scales, dtype=np.float16))
    out = channelwise_int_decompress_device(scales, codes, packet.shape, packet.bits,
                                            torch.float64)
    return _download(out)


def serialize_channel_int(packet: ChannelIntPacket) -> bytes:
    header = pack_header(FORMAT_CODE_CHANNEL_INT, packet.bits, 0, packet.shape)
    return header + packet.scales.astype("<f2").tobytes() + packet.code_stream


def deserialize_channel_int(data: bytes) -> ChannelIntPacket:
    format_code, bits, _, shape, offset = unpack_header(data)
    if format_code != FORMAT_CODE_CHANNEL_INT:
        raise MalformedHeader(f"format code {format_code:#x} is not channel INT")
    if not 2 <= bits <= 8:
        raise MalformedHeader(f"channel INT bit width {bits} outside [2, 8]")
    channels = shape[-1]
    n = int(np.prod(shape, dtype=np.int64))
    scale_end = offset + 2 * channels
    code_bytes = packed_nbytes(n, bits)
    if len(data) < scale_end + code_bytes:
        raise TruncatedStream("channel INT payload shorter than declared shape")
    return ChannelIntPacket(shape=shape, bits=bits,
                            scales=np.frombuffer(data, "<f2", count=channels, offset=offset).copy(),
                            code_stream=data[scale_end:scale_end + code_bytes])
