"""Deterministic parity inputs shared by the golden generator and the tests.

Every generator returns float64 values that are exactly representable in
the dtype named by the case (bf16 / f16 / f32), so the same bytes can be fed
to the reference (float64), to the oracle, and to the CUDA kernels.
"""

from __future__ import annotations

import numpy as np

from paper_2411_09510_b200.synth import bf16_round, gaussian_with_outliers

# schemes covered by the exhaustive digest sweep
REGISTRY_ELEMENTS = ["fp4_e2m1", "fp5_e2m2", "fp5_e3m1", "fp5_e1m3", "fp4_e1m2",
                     "fp3_e1m1", "fp2_e1m0", "int3", "int4", "int5"]
EXTENSION_ELEMENTS = ["fp6_e2m3", "fp6_e3m2", "int8", "fp3_e2m0", "fp8_e4m3", "fp8_e5m2"]
BLOCKS = [8, 16, 32, 64]
ODD_BLOCKS = [1, 7, 24, 100, 256, 512]
SCALES = ["e8m0", "e5m0", "e4m0", "e6m0", "e7m0"]


def sweep_schemes():
    out = []
    for el in REGISTRY_ELEMENTS + EXTENSION_ELEMENTS:
        for b in BLOCKS:
            out.append(f"{el}:{b}:e8m0")
        out.append(f"{el}:32:e5m0")
        out.append(f"{el}:16:e4m0")
    for el in ["fp4_e2m1", "fp5_e2m2", "int8", "fp6_e3m2"]:
        for b in ODD_BLOCKS:
            out.append(f"{el}:{b}:e8m0")
        for sc in SCALES:
            out.append(f"{el}:32:{sc}")
    # dedupe, keep order
    seen, res = set(), []
    for s in out:
        if s not in seen:
            seen.add(s)
            res.append(s)
    return res


def all_bf16(seed: int = 0) -> np.ndarray:
    """Every finite bfloat16 value (both zeros included), shuffled so that
    blocks mix magnitudes; length 65,280 (not a multiple of 64: tail block)."""
    bits = np.arange(1 << 16, dtype=np.uint32)
    f = (bits << 16).view(np.float32)
    f = f[np.isfinite(f)]
    f = f[np.random.default_rng(seed).permutation(f.size)]
    f = f[: f.size - 17]  # ragged tail
    return f.astype(np.float64)


def all_bf16_sorted_blocks() -> np.ndarray:
    """Finite bf16 values sorted by magnitude: neighbouring values share a
    block, so the scale is set by a close neighbour and every element code
    (incl. midpoint ties) is exercised."""
    bits = np.arange(1 << 16, dtype=np.uint32)
    f = (bits << 16).view(np.float32)
    f = f[np.isfinite(f)]
    order = np.argsort(np.abs(f), kind="stable")
    return f[order].astype(np.float64)


def gauss_bf16(n: int, seed: int) -> np.ndarray:
    return bf16_round(gaussian_with_outliers(np.random.default_rng(seed), (n,))).astype(np.float64)


def gauss_f32(n: int, seed: int) -> np.ndarray:
    return gaussian_with_outliers(np.random.default_rng(seed), (n,)).astype(np.float64)


def gauss_f16(n: int, seed: int) -> np.ndarray:
    x = gaussian_with_outliers(np.random.default_rng(seed), (n,), magnification=30.0)
    return x.astype(np.float16).astype(np.float64)


def extremes_f32(n: int, seed: int) -> np.ndarray:
    """f32 values over the whole exponent range (subnormals to near FLT_MAX),
    random signs, signed zeros and all-zero blocks sprinkled in."""
    rng = np.random.default_rng(seed)
    e = rng.integers(-149, 128, size=n)
    m = rng.random(n) + 1.0
    x = np.ldexp(m, e).astype(np.float32).astype(np.float64)
    x[~np.isfinite(x)] = 1.0
    x *= np.where(rng.random(n) < 0.5, -1.0, 1.0)
    # blocks of locally similar magnitude, so scales are not all clamped
    x = x[np.argsort(np.abs(x), kind="stable")]
    perm = rng.permutation(n // 64)
    x = x[: (n // 64) * 64].reshape(-1, 64)[perm].ravel()
    x[rng.random(x.size) < 0.02] = 0.0
    x[rng.random(x.size) < 0.02] = -0.0
    x[128:192] = 0.0
    x[256:320] = -0.0
    return x


def random_streams(nbytes_scale: int, nbytes_elem: int, seed: int):
    rng = np.random.default_rng(seed)
    return (rng.integers(0, 256, nbytes_scale, dtype=np.uint8).tobytes(),
            rng.integers(0, 256, nbytes_elem, dtype=np.uint8).tobytes())


CASES = {
    # name -> (generator, dtype the kernels are fed)
    "all_bf16": (lambda: all_bf16(0), "bf16"),
    "sorted_bf16": (all_bf16_sorted_blocks, "bf16"),
    "gauss_bf16_4099": (lambda: gauss_bf16(4099, 3), "bf16"),
    "gauss_f32_5003": (lambda: gauss_f32(5003, 4), "f32"),
    "gauss_f16_3001": (lambda: gauss_f16(3001, 5), "f16"),
    "extremes_f32_8192": (lambda: extremes_f32(8192, 6), "f32"),
}

LARGE_SHAPE = (2048, 4096)
LARGE_SCHEMES = ["fp4_e2m1:32:e8m0", "fp4_e2m1:16:e8m0", "fp4_e2m1:64:e8m0",
                 "fp5_e2m2:32:e8m0", "fp6_e2m3:32:e8m0", "int8:32:e8m0",
                 "fp4_e2m1:32:e5m0"]


# ---------------------------------------------------------------------------
# comparison codecs (mx/baselines.py): shaped cases, channels = last dim
# ---------------------------------------------------------------------------


def ties_bf16(rows: int, cols: int, seed: int) -> np.ndarray:
    """Few distinct magnitudes (TopK ties, broken toward the lower index),
    an all-zero and an all-(-0) channel, and a channel whose scale is
    exactly 1 at 4 bits (max 7) so x/scale lands on .5 ties."""
    rng = np.random.default_rng(seed)
    x = rng.choice(np.array([0.0, 0.5, -0.5, 1.0, -1.0, 1.5, 2.0, -2.0, 3.0, -3.0]),
                   size=(rows, cols))
    x[:, 5] = 0.0
    x[:, 9] = -0.0
    x[:, 3] = rng.choice(np.array([0.5, 1.5, 2.5, -3.5, -0.5, 4.5]), size=rows)
    x[0, 3] = 7.0
    return x


def wide_range_f32(rows: int, cols: int, seed: int) -> np.ndarray:
    """Per-channel magnitudes from 1e-9 to 1e6: f16 scales that are
    subnormal, normal and (at low bit widths) overflow to inf."""
    rng = np.random.default_rng(seed)
    mag = 10.0 ** rng.uniform(-9, 6, size=cols)
    x = rng.standard_normal((rows, cols)) * mag
    return x.astype(np.float32).astype(np.float64)


BASELINE_CASES = {
    "gauss_bf16_64x256": (lambda: gauss_bf16(64 * 256, 11).reshape(64, 256), "bf16"),
    "gauss_f32_33x100": (lambda: gauss_f32(3300, 12).reshape(33, 100), "f32"),
    "gauss_f16_777": (lambda: gauss_f16(777, 13), "f16"),
    "ties_bf16_48x64": (lambda: ties_bf16(48, 64, 14), "bf16"),
    "wide_f32_16x40": (lambda: wide_range_f32(16, 40, 15), "f32"),
    "prefill_bf16_2048x4096": (
        lambda: bf16_round(gaussian_with_outliers(np.random.default_rng(0), (2048, 4096)))
        .astype(np.float64), "bf16"),
}


def baseline_case(name: str) -> np.ndarray:
    return BASELINE_CASES[name][0]()
