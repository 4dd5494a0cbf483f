"""GPU evaluators for the compression-scheme search (mx/search.py:230-248).

The reference scores a candidate scheme by the relative Frobenius error of a
seeded tensor-parallel reduction (``make_simulation_evaluator`` ->
``tpsim.simulate_reduction(cfg).rel_frob_err * 100``), recomputing the
inputs, the partial products and a numpy codec round trip per candidate.
Here the per-rank partials are computed once and stay resident on the
device; each candidate is one K1 quantise + one exact float64 decode per
rank (the reference's ``decoded[r]``), the float64 rank-order sum and the
error norms -- all on the GPU, one host read per candidate (or one per batch
with :meth:`DeviceReductionEvaluator.evaluate_many`).

The evaluators are plain callables ``scheme -> degradation %``, so they
plug straight into the reference's own selection code::

    import mxcomm.search as ref_search
    from paper_2411_09510_b200.search import make_simulation_evaluator
    ref_search.run_grid(ref_search.SearchConfig(...), make_simulation_evaluator())

:func:`make_activation_evaluator` scores candidates on real activation
dumps (per-rank row-parallel partials saved from a model), the ablation
path the reference's metric tables stand in for.
"""

from __future__ import annotations

import math

import numpy as np

from . import _native
from .codec import compress_tensor_device, decompress_tensor_device
from .errors import MinimumDegreeTwo, ShapeMismatch
from .formats import SchemeDescriptor, parse_scheme
from .tp import ReductionReport, TPConfig, UNCOMPRESSED_VALUE_BYTES, generate_inputs, shard_rowwise


def _torch():
    import torch

    return torch


class DeviceReductionEvaluator:
    """Score MX schemes on fixed per-rank partials kept on the GPU.

    ``partials``: one array / tensor per rank (any float dtype; quantised as
    float32 like the reference's ``x_shard @ w_shard`` partials,
    mx/tpsim.py:263).  ``quantize_own`` as TPConfig (mx/tpsim.py:155): False
    keeps rank 0's partial exact.  ``evaluator(scheme)`` returns
    ``rel_frob_err * 100`` (mx/search.py:243-246); :meth:`report` returns the
    full :class:`ReductionReport` (mx/tpsim.py:272-302)."""

    def __init__(self, partials, quantize_own: bool = True, device=None):
        torch = _torch()
        _native.require_cuda()
        if len(partials) < 2:
            raise MinimumDegreeTwo(f"degree {len(partials)} < 2")
        dev = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        ts = []
        for p in partials:
            t = p if hasattr(p, "is_cuda") else torch.from_numpy(np.ascontiguousarray(p))
            ts.append(t.to(dev, torch.float32).contiguous())
        self.shape = tuple(ts[0].shape)
        if any(tuple(t.shape) != self.shape for t in ts):
            raise ShapeMismatch("every rank's partial must have the same shape")
        self.partials = [t.reshape(-1) for t in ts]
        for r, t in enumerate(self.partials):  # once, so K1 needs no per-call sync
            if not bool(torch.isfinite(t).all().item()):
                from .errors import NonFiniteInput

                bad = int(torch.nonzero(~torch.isfinite(t))[0].item())
                raise NonFiniteInput(f"non-finite value in rank {r}'s partial "
                                     f"(flat index {bad})", block_index=None)
        self.degree = len(ts)
        self.quantize_own = quantize_own
        self.device = dev
        # exact reference sum: float64, rank order (mx/tpsim.py:275-281)
        ref = torch.zeros(self.partials[0].numel(), dtype=torch.float64, device=dev)
        for t in self.partials:
            ref += t.double()
        self.ref = ref
        self._ref_norm = torch.linalg.vector_norm(ref)
        self._ref_sq = torch.sum(ref * ref)

    @staticmethod
    def _scheme(scheme) -> SchemeDescriptor:
        return scheme if isinstance(scheme, SchemeDescriptor) else parse_scheme(str(scheme))

    def _reduce(self, sch):
        """Device float64 error vector and the per-worker error budget."""
        torch = _torch()
        red = torch.zeros_like(self.ref)
        per = torch.zeros_like(self.ref)
        payload = None
        for r, p in enumerate(self.partials):
            if self.quantize_own or r != 0:
                dct = compress_tensor_device(p, sch, check_finite=False)
                if payload is None:
                    payload = dct.scale.numel() + dct.elements.numel()
                dec = decompress_tensor_device(dct, torch.float64).reshape(-1)
            else:
                dec = p.double()
            red += dec
            per += (dec - p.double()).abs()
        if payload is None:  # quantize_own=False with one quantised rank at least
            payload = 0
        return red - self.ref, per, payload

    def __call__(self, scheme) -> float:
        torch = _torch()
        err, _, _ = self._reduce(self._scheme(scheme))
        en = torch.linalg.vector_norm(err)
        v = torch.where(en == 0, torch.zeros_like(en), en / self._ref_norm)
        return float(v.item()) * 100.0

    def evaluate_many(self, schemes) -> list:
        """Score a batch of candidates with ONE host read at the end."""
        torch = _torch()
        vals = []
        for s in schemes:
            err, _, _ = self._reduce(self._scheme(s))
            en = torch.linalg.vector_norm(err)
            vals.append(torch.where(en == 0, torch.zeros_like(en), en / self._ref_norm))
        if not vals:
            return []
        return [float(v) * 100.0 for v in torch.stack(vals).cpu().tolist()]

    def report(self, scheme, padding: int = 0) -> ReductionReport:
        """The reference's ReductionReport for this candidate, with the
        per-worker error-budget check (mx/tpsim.py:284-288)."""
        from .codec import header_nbytes

        torch = _torch()
        sch = self._scheme(scheme)
        err, per, payload = self._reduce(sch)
        tol = 1e-9 * (self.ref.abs() + 1.0)
        ok = bool(torch.all(err.abs() <= per + tol).item())
        if not ok:
            raise AssertionError("summed error exceeded per-worker error budget")
        en = float(torch.linalg.vector_norm(err).item())
        rn = float(self._ref_norm.item())
        esq = float(torch.sum(err * err).item())
        rsq = float(self._ref_sq.item())
        sqnr = math.inf if esq == 0.0 else (
            -math.inf if rsq == 0.0 else 10.0 * math.log10(rsq / esq))
        n = self.ref.numel()
        return ReductionReport(
            degree=self.degree, scheme=str(sch), rel_frob_err=0.0 if en == 0.0 else en / rn,
            max_abs_err=float(err.abs().max().item()), sqnr_db=sqnr,
            bytes_compressed=(self.degree - 1) * (header_nbytes(len(self.shape)) + payload),
            bytes_uncompressed=(self.degree - 1) * n * UNCOMPRESSED_VALUE_BYTES,
            padding=padding)


def simulation_partials(degree: int = 2, seed: int = 0, input_shape=(1, 64, 512),
                        weight_shape=(512, 512)):
    """The reference evaluator's per-rank float32 partials
    ``x[..., rows_r] @ shard_r`` from its seeded inputs (mx/tpsim.py:218-265),
    computed with numpy exactly as the reference does; -> (partials, padding)."""
    cfg = TPConfig(degree=degree, scheme=None, seed=seed, input_shape=tuple(input_shape),
                   weight_shape=tuple(weight_shape))
    x, w = generate_inputs(cfg)
    x = np.asarray(x, dtype=np.float32)
    w = np.asarray(w, dtype=np.float32)
    shards, padding = shard_rowwise(w, degree)
    if padding:
        x = np.pad(x, [(0, 0)] * (x.ndim - 1) + [(0, padding)])
    rows = shards[0].shape[0]
    return [x[..., r * rows:(r + 1) * rows] @ shards[r] for r in range(degree)], padding


def make_simulation_evaluator(degree: int = 2, seed: int = 0, input_shape=(1, 64, 512),
                              weight_shape=(512, 512), partials=None):
    """mx/search.py:230-248 on the GPU: ``evaluate(scheme)`` = the seeded
    reduction's relative Frobenius error in percent.  ``partials`` replays
    precomputed per-rank products (BLAS results depend on the host CPU, so
    parity tests pass the reference's own)."""
    if partials is None:
        partials, _ = simulation_partials(degree, seed, input_shape, weight_shape)
    elif len(partials) != degree:
        raise ShapeMismatch(f"{len(partials)} partials for degree {degree}")
    return DeviceReductionEvaluator(partials)


def load_activation_dump(path):
    """Per-rank row-parallel partials from a dump: ``.npy`` / ``.pt`` holding
    one array of shape [ranks, ...], or ``.npz`` with one array per rank
    (sorted by key)."""
    if str(path).endswith(".npz"):
        with np.load(path) as z:
            return [z[k] for k in sorted(z.files)]
    if str(path).endswith(".pt"):
        t = _torch().load(path, map_location="cpu")
        return list(t) if not isinstance(t, (list, tuple)) else list(t)
    a = np.load(path)
    return [a[i] for i in range(a.shape[0])]


def make_activation_evaluator(dump, quantize_own: bool = True):
    """Score candidates on REAL activations: ``dump`` is a list of per-rank
    partials (arrays / tensors, e.g. captured at a model's o_proj or
    down_proj) or a path for :func:`load_activation_dump`."""
    partials = load_activation_dump(dump) if isinstance(dump, (str, bytes)) or hasattr(
        dump, "__fspath__") else list(dump)
    return DeviceReductionEvaluator(partials, quantize_own=quantize_own)
