"""CPU restatement of the reference's comparison codecs (mx/baselines.py).

TEST INFRASTRUCTURE ONLY -- the checker for the sm_100a TopK / channel-INT
kernels; same import rules as ``oracle/mx_oracle.py``.  Pinned against
``tests/golden/baselines.json`` (made by running the real reference,
``tests/golden/make_golden_baselines.py``) in ``tests/test_oracle_golden.py``.

Restated, not copied:

* channel-wise INT (mx/baselines.py:138-168): the per-channel scale is the
  f16 rounding of ``max|x| / (2^(b-1)-1)`` (float64 division); the level is
  round-half-even of ``x / scale`` written here as an exact integer
  comparison against ``(k + 1/2) * scale`` (every such product is exact in
  float64 for f16 scales and levels < 2^8), clamped to +-qmax; sign-magnitude
  codes (sign only for levels < 0), LSB-first packed (mx/bitpack.py:22-34);
  decode = level * scale in float64 (mx/baselines.py:171-178).
* TopK (mx/baselines.py:95-135): K = floor((2n/F - header) / 6)
  (``topk_budget`` 88-92); keep the K largest |x|, ties toward the lower
  index, written here as a lexicographic sort on (-|x|, index); indices
  ascending as u32, values as f16; decode scatters into zeros.
"""

from __future__ import annotations

import numpy as np

from oracle.mx_oracle import pack, unpack

HEADER_FIXED = 20  # MXC1 header: 20 + 8 * ndim bytes (mx/codec.py:287-289)


def header_nbytes(ndim: int) -> int:
    return HEADER_FIXED + 8 * ndim


def chanint_compress(x, bits: int):
    """Returns (scales float16[C], codes uint8[n], code_stream bytes)."""
    a = np.asarray(x, dtype=np.float64)
    if a.ndim < 1:
        a = a.reshape(1)
    qmax = (1 << (bits - 1)) - 1
    cols = a.reshape(-1, a.shape[-1])
    with np.errstate(over="ignore"):
        s16 = (np.abs(cols).max(axis=0) / qmax).astype(np.float16)
    s = s16.astype(np.float64)
    mag = np.abs(cols)
    lev = np.zeros(cols.shape, dtype=np.int64)
    ok = (s > 0) & np.isfinite(s)
    with np.errstate(divide="ignore", invalid="ignore"):
        k = np.where(ok, np.floor(mag / np.where(ok, s, 1.0)), 0).astype(np.int64)
    # exact correction of floor(mag/s) and the half-way test
    k = np.where(ok & (k * s > mag), k - 1, k)
    k = np.where(ok & ((k + 1) * s <= mag), k + 1, k)
    half = (k + 0.5) * s
    up = (mag > half) | ((mag == half) & (k % 2 == 1))
    lev = np.where(ok, np.minimum(k + up, qmax), 0)
    neg = (cols < 0) & (lev > 0)
    codes = (lev | np.where(neg, 1 << (bits - 1), 0)).astype(np.uint8).ravel()
    return s16, codes, pack(codes, bits)


def chanint_decompress(scales16, code_stream: bytes, shape, bits: int) -> np.ndarray:
    n = int(np.prod(shape, dtype=np.int64)) if len(shape) else 1
    codes = unpack(code_stream, n, bits).astype(np.int64)
    mag = (codes & ((1 << (bits - 1)) - 1)).astype(np.float64)
    sgn = np.where(codes >> (bits - 1), -1.0, 1.0)
    with np.errstate(invalid="ignore"):
        return ((sgn * mag).reshape(-1, shape[-1]) * scales16.astype(np.float64)).reshape(shape)


def topk_budget(n: int, ndim: int, factor: float) -> int:
    return int((n * 2 / factor - header_nbytes(ndim)) // 6)


def topk_compress(x, factor=None, k=None):
    """Returns (indices uint32[K] ascending, values float16[K])."""
    a = np.asarray(x, dtype=np.float64)
    flat = a.ravel()
    if k is None:
        k = topk_budget(flat.size, a.ndim, factor)
    k = min(int(k), flat.size)
    order = np.lexsort((np.arange(flat.size), -np.abs(flat)))[:k]
    idx = np.sort(order)
    with np.errstate(over="ignore"):
        vals = flat[idx].astype(np.float16)
    return idx.astype(np.uint32), vals


def topk_decompress(indices, values, shape) -> np.ndarray:
    n = int(np.prod(shape, dtype=np.int64)) if len(shape) else 1
    out = np.zeros(n)
    out[np.asarray(indices, dtype=np.int64)] = np.asarray(values).astype(np.float64)
    return out.reshape(shape)
