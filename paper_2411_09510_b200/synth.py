"""Synthetic activation generator (restates mx/synth.py:17-29).

Real row-parallel partial sums are roughly Gaussian with a sparse population
of large-magnitude outliers; that population is what makes coarse
absolute-max scaling lossy and fine-grained MX blocks worthwhile.
"""

from __future__ import annotations

import numpy as np

OUTLIER_FRACTION = 0.01  # mx/synth.py:13
OUTLIER_MAGNIFICATION = 100.0  # mx/synth.py:14


def gaussian_with_outliers(rng: np.random.Generator, shape, fraction=OUTLIER_FRACTION,
                           magnification=OUTLIER_MAGNIFICATION, dtype=np.float32):
    """N(0,1) draws; a Bernoulli(``fraction``) subset is multiplied by
    ``magnification``.  Draw order (normals, then uniforms) is kept so the
    same seed yields the reference's tensor bit for bit."""
    base = rng.standard_normal(shape)
    if fraction > 0:
        hit = rng.random(shape) < fraction
        base = np.where(hit, base * magnification, base)
    return base.astype(dtype)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """float32 values rounded (RNE) to the nearest bfloat16, returned as
    float32 -- the exact values a bf16 partial-sum tensor holds."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).reshape(np.shape(x))


def rank_partials(shape, nranks: int, seed: int = 0):
    """Per-rank bf16-valued partial sums, seeds ``seed+r``."""
    return [bf16_round(gaussian_with_outliers(np.random.default_rng(seed + r), shape))
            for r in range(nranks)]
