"""CPU restatement of the mxcomm compressed-collective hot path.

TEST INFRASTRUCTURE ONLY.  This module is the *checker* for the sm_100a
kernels: it may be imported by ``tests/``, by ``__graft_entry__.smoke()`` and
by the ``cpu_baseline`` / ``--impl reference`` legs of ``bench.py``.  The
product package ``paper_2411_09510_b200`` never imports it, and nothing here
is ever on a measured GPU path.

It restates, in plain numpy, the algorithm of the reference package
``mxcomm`` (``/root/reference/pkg/src/mxcomm``, abbreviated ``mx/`` below):

* element grids / emax              -- mx/formats.py:189-212
* scale-format exponent range        -- mx/formats.py:116-128
* block quantiser                    -- mx/codec.py:140-172 (+ _round_to_grid 127-137)
* LSB-first fixed-width bit packing  -- mx/bitpack.py:22-58
* block dequantiser                  -- mx/codec.py:175-188
* compress/decompress_tensor         -- mx/codec.py:238-284
* non-finite detection               -- mx/codec.py:191-199
* one-shot compressed all-reduce     -- mx/netbench.py:323-334 (fp32, rank order, +0 init)
* two-shot (reduce-scatter/requantise/all-gather) -- NOT in the reference;
  restated here from the same codec calls (SURVEY.md §8(c) "restatement").

Parity is PINNED: ``tests/golden/`` holds byte streams and SHA-256 digests
produced by running the real reference in the build container
(``tests/golden/make_golden.py``); ``tests/test_oracle_golden.py`` checks this
restatement against every one of them before any GPU result is compared with
it.

The rounding is written differently from the reference (closed-form
floor/fraction on the exact float64 value instead of ``searchsorted`` over
midpoints) -- the golden vectors prove the two agree, including the
"ties to the even grid index" rule for zero-mantissa formats.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

# ---------------------------------------------------------------------------
# Scheme description (independent of the product package on purpose)
# ---------------------------------------------------------------------------

_FLOAT, _INT = "float", "int"

# element name -> (kind, exponent bits, mantissa bits); registry order of
# mx/formats.py:218-229 first, then the BASELINE.json sweep extensions.
ELEMENTS = {
    "fp4_e2m1": (_FLOAT, 2, 1),
    "fp5_e2m2": (_FLOAT, 2, 2),
    "fp5_e3m1": (_FLOAT, 3, 1),
    "fp5_e1m3": (_FLOAT, 1, 3),
    "fp4_e1m2": (_FLOAT, 1, 2),
    "fp3_e1m1": (_FLOAT, 1, 1),
    "fp2_e1m0": (_FLOAT, 1, 0),
    "int3": (_INT, 0, 2),
    "int4": (_INT, 0, 3),
    "int5": (_INT, 0, 4),
    # extensions (constructible in the reference, absent from its registry)
    "fp6_e2m3": (_FLOAT, 2, 3),
    "fp6_e3m2": (_FLOAT, 3, 2),
    "int8": (_INT, 0, 7),
    "fp3_e2m0": (_FLOAT, 2, 0),
    "fp8_e4m3": (_FLOAT, 4, 3),
    "fp8_e5m2": (_FLOAT, 5, 2),
}


@dataclass(frozen=True)
class OScheme:
    kind: str
    ebits: int
    mbits: int
    block: int
    kbits: int

    # -- element format -------------------------------------------------
    @property
    def bits(self) -> int:
        return 1 + self.ebits + self.mbits

    @property
    def elem_bias(self) -> int:  # mx/formats.py:89-94
        return 0 if self.kind == _INT else (1 << (self.ebits - 1)) - 1

    @property
    def grid(self) -> np.ndarray:
        return element_grid(self.kind, self.ebits, self.mbits)

    @property
    def grid_max(self) -> float:
        return float(self.grid[-1])

    @property
    def emax(self) -> int:  # mx/formats.py:208-212
        return math.frexp(self.grid_max)[1] - 1

    # -- scale format ---------------------------------------------------
    @property
    def scale_bias(self) -> int:  # mx/formats.py:116-118
        return (1 << (self.kbits - 1)) - 1

    @property
    def s_min(self) -> int:  # mx/formats.py:120-123
        return 1 - self.scale_bias

    @property
    def s_max(self) -> int:  # mx/formats.py:125-128
        return (1 << self.kbits) - 1 - self.scale_bias

    @property
    def name(self) -> str:
        for nm, spec in ELEMENTS.items():
            if spec == (self.kind, self.ebits, self.mbits):
                return f"{nm}:{self.block}:e{self.kbits}m0"
        return f"{self.kind}{self.ebits}.{self.mbits}:{self.block}:e{self.kbits}m0"


def scheme(spec: str) -> OScheme:
    """``"fp4_e2m1:32:e8m0"`` -> OScheme (extension element names accepted)."""
    el, blk, sc = spec.split(":")
    kind, e, m = ELEMENTS[el]
    assert sc[0] == "e" and sc.endswith("m0")
    return OScheme(kind, e, m, int(blk), int(sc[1:-2]))


def element_grid(kind: str, ebits: int, mbits: int) -> np.ndarray:
    """Ascending non-negative magnitudes (mx/formats.py:189-205).

    Closed form: index ``i = e_field << m | mant``; e_field 0 is subnormal
    ``mant * 2^(1-bias-m)``, otherwise ``(2^m + mant) * 2^(e_field-bias-m)``.
    INTn (sign-magnitude) is ``0 .. 2^(n-1)-1``.
    """
    n = 1 << (ebits + mbits)
    idx = np.arange(n, dtype=np.int64)
    if kind == _INT:
        return idx.astype(np.float64)
    bias = (1 << (ebits - 1)) - 1
    ef = idx >> mbits
    mant = idx & ((1 << mbits) - 1)
    sig = np.where(ef > 0, mant + (1 << mbits), mant)
    exp = np.maximum(ef, 1) - bias - mbits
    return np.ldexp(sig.astype(np.float64), exp)


# ---------------------------------------------------------------------------
# Quantiser (mx/codec.py:140-172)
# ---------------------------------------------------------------------------


def shared_exponent(amax: np.ndarray, sch: OScheme) -> np.ndarray:
    """Per-block unbiased shared exponent, clamped (mx/codec.py:155-161).

    floor(log2 amax) - emax, bumped by one when the scaled maximum would
    still exceed the top grid value, then clamped to the scale range.
    Zero blocks get an arbitrary value (callers mask them).
    """
    safe = np.where(amax > 0, amax, 1.0)
    flog = np.frexp(safe)[1].astype(np.int64) - 1
    s = flog - sch.emax
    s = s + (np.ldexp(safe, -s) > sch.grid_max)
    return np.clip(s, sch.s_min, sch.s_max)


def grid_index(mag: np.ndarray, sch: OScheme) -> np.ndarray:
    """Nearest grid index of non-negative exact magnitudes, saturating,
    exact midpoints to the EVEN index (mx/codec.py:127-137).

    Closed form used by the kernels too: with lo = 1-bias (float) or
    lo = y = n-1 (int), q = max(floor(log2 a), lo), the grid spacing at
    ``a`` is 2^(q-y) and ``index = floor(a/2^(q-y)) + ((q-lo) << y)`` plus a
    round-up on fractions above 1/2, or exactly 1/2 with an odd index.
    """
    y = sch.mbits
    lo = (1 - sch.elem_bias) if sch.kind == _FLOAT else sch.mbits
    a = np.minimum(mag, sch.grid_max)
    pos = a > 0
    flog = np.frexp(np.where(pos, a, 1.0))[1].astype(np.int64) - 1
    q = np.where(pos, np.maximum(flog, lo), lo)
    t = np.ldexp(a, -(q - y))  # exact
    r0 = np.floor(t)
    frac = t - r0
    base = r0.astype(np.int64) + ((q - lo) << y)
    up = (frac > 0.5) | ((frac == 0.5) & ((base & 1) == 1))
    return base + up


def quantize(flat: np.ndarray, sch: OScheme):
    """Block-quantise a flat float64 vector -> (stored u8[nb], codes u8[n])."""
    flat = np.asarray(flat, dtype=np.float64).ravel()
    n = flat.size
    nb = -(-n // sch.block)
    padded = np.zeros(nb * sch.block)
    padded[:n] = flat
    blocks = padded.reshape(nb, sch.block)
    amax = np.abs(blocks).max(axis=1) if nb else np.zeros(0)
    zero = amax == 0
    s = shared_exponent(amax, sch)
    scaled = np.ldexp(blocks, -s[:, None])
    idx = grid_index(np.abs(scaled), sch)
    sign = np.signbit(scaled).astype(np.int64)
    codes = (sign << (sch.bits - 1)) | idx
    codes[zero] = 0
    stored = np.where(zero, 0, s + sch.scale_bias)
    return stored.astype(np.uint8), codes.reshape(-1)[:n].astype(np.uint8)


# ---------------------------------------------------------------------------
# Bit packing (mx/bitpack.py:22-58): value i at bit i*w, LSB first
# ---------------------------------------------------------------------------


def pack(codes: np.ndarray, width: int) -> bytes:
    """Groups of 8 codes form one ``8*width``-bit little-endian integer,
    i.e. exactly ``width`` bytes; the last group is zero-padded."""
    c = np.asarray(codes, dtype=np.uint64).ravel()
    n = c.size
    if n == 0:
        return b""
    g = -(-n // 8)
    buf = np.zeros(g * 8, dtype=np.uint64)
    buf[:n] = c
    buf = buf.reshape(g, 8)
    word = np.zeros(g, dtype=np.uint64)
    for j in range(8):
        word |= buf[:, j] << np.uint64(j * width)
    out = word.view(np.uint8).reshape(g, 8)[:, :width]  # little-endian host
    return out.tobytes()[: (n * width + 7) // 8]


def unpack(data: bytes, count: int, width: int) -> np.ndarray:
    need = (count * width + 7) // 8
    if len(data) < need:
        raise ValueError("truncated stream")
    g = -(-count // 8)
    raw = np.zeros(g * width, dtype=np.uint8)
    raw[:need] = np.frombuffer(data, dtype=np.uint8, count=need)
    words = np.zeros((g, 8), dtype=np.uint8)
    words[:, :width] = raw.reshape(g, width)
    word = words.view(np.uint64).ravel()
    mask = np.uint64((1 << width) - 1)
    out = np.empty((g, 8), dtype=np.uint8)
    for j in range(8):
        out[:, j] = (word >> np.uint64(j * width)) & mask
    return out.ravel()[:count]


# ---------------------------------------------------------------------------
# Dequantiser (mx/codec.py:175-188)
# ---------------------------------------------------------------------------


def dequantize(stored: np.ndarray, codes: np.ndarray, n: int, sch: OScheme,
               dtype=np.float64) -> np.ndarray:
    grid = sch.grid
    lut = np.concatenate([grid, -grid])
    nb = stored.size
    full = np.zeros(nb * sch.block, dtype=np.int64)
    full[:n] = codes
    vals = lut[full].reshape(nb, sch.block)
    st = stored.astype(np.int64)
    factor = np.where(st == 0, 0.0, np.ldexp(1.0, st - sch.scale_bias))
    return (vals * factor[:, None]).astype(dtype).ravel()[:n]


# ---------------------------------------------------------------------------
# Tensor-level codec (mx/codec.py:238-284)
# ---------------------------------------------------------------------------


class NonFinite(ValueError):
    def __init__(self, block_index: int):
        super().__init__(f"non-finite input in block {block_index}")
        self.block_index = block_index


def first_nonfinite_block(flat: np.ndarray, block: int):
    """mx/codec.py:191-199: block index of the first NaN/Inf, else None."""
    bad = np.flatnonzero(~np.isfinite(flat))
    return None if bad.size == 0 else int(bad[0]) // block


def compress(arr, sch: OScheme):
    """-> (scale_stream bytes, element_stream bytes); raises NonFinite."""
    flat = np.asarray(arr, dtype=np.float64).ravel()
    b = first_nonfinite_block(flat, sch.block)
    if b is not None:
        raise NonFinite(b)
    stored, codes = quantize(flat, sch)
    return pack(stored, sch.kbits), pack(codes, sch.bits)


def decompress(scale_stream: bytes, element_stream: bytes, n: int, sch: OScheme,
               dtype=np.float64) -> np.ndarray:
    nb = -(-n // sch.block)
    stored = unpack(scale_stream, nb, sch.kbits)
    codes = unpack(element_stream, n, sch.bits)
    return dequantize(stored, codes, n, sch, dtype)


def roundtrip_f32(arr, sch: OScheme) -> np.ndarray:
    """decompress(compress(x), float32): what a rank contributes."""
    flat = np.asarray(arr, dtype=np.float64).ravel()
    stored, codes = quantize(flat, sch)
    return dequantize(stored, codes, flat.size, sch, np.float32)


# ---------------------------------------------------------------------------
# Collectives (mx/netbench.py:323-334)
# ---------------------------------------------------------------------------


def allreduce_oneshot(partials, sch: OScheme) -> np.ndarray:
    """Every rank's partial is quantised (own included, mx/netbench.py:323),
    decoded to float32 and summed from +0.0 in rank order (332-334)."""
    acc = np.zeros(np.asarray(partials[0]).size, dtype=np.float32)
    for p in partials:
        acc += roundtrip_f32(p, sch)
    return acc


def twoshot_chunks(n: int, nranks: int, block: int, align: int = 8):
    """Chunk boundaries of the two-shot path: N contiguous pieces whose
    length is a multiple of ``align*block`` (blocks never straddle a chunk,
    so per-chunk quantisation equals whole-tensor quantisation)."""
    unit = align * block
    per = -(-n // nranks)
    per = -(-per // unit) * unit
    return [(min(j * per, n), min((j + 1) * per, n)) for j in range(nranks)]


def allreduce_twoshot(partials, sch: OScheme, chunk_align: int = 8) -> np.ndarray:
    """Reduce-scatter of quantised chunks, fp32 rank-order sum per chunk,
    requantise the sum, all-gather, decode (restatement; not in the reference).
    Like every one-shot output value, the decoded value is accumulated into a
    +0.0 float32 accumulator (mx/netbench.py:332), so a -0 code yields +0."""
    flats = [np.asarray(p, dtype=np.float64).ravel() for p in partials]
    n = flats[0].size
    out = np.zeros(n, dtype=np.float32)
    for lo, hi in twoshot_chunks(n, len(flats), sch.block, chunk_align):
        if hi <= lo:
            continue
        acc = np.zeros(hi - lo, dtype=np.float32)
        for f in flats:
            acc += roundtrip_f32(f[lo:hi], sch)
        out[lo:hi] = np.float32(0.0) + roundtrip_f32(acc, sch)
    return out


def to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """float32 -> bfloat16 bit patterns, round-to-nearest-even."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    nan = np.isnan(x)
    r = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    r = np.where(nan.ravel() if r.ndim == 1 else nan, 0x7FC0, r)
    return r.astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)
