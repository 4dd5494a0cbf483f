"""CPU codec backend built on the oracle -- TEST DOUBLE ONLY.

Plugs into ``paper_2411_09510_b200.collective.CompressedAllReduce`` in place
of the sm_100a ``NativeBackend`` so the collective's orchestration (buffer
layout, chunking, all_to_all / all_gather order, rank-order reduction) can
be exercised with ``gloo`` on CPU.  The shard layout itself comes from the
real library (``mx_shard_layout`` is host-only and needs no GPU).
"""

import numpy as np
import torch

from oracle import mx_oracle as O
from paper_2411_09510_b200 import _native


class OracleBackend:
    def __init__(self, scheme):
        self.scheme = scheme
        self.cs = scheme.to_c()
        self.o = O.scheme(scheme.name) if scheme.element.name in O.ELEMENTS else O.OScheme(
            "float" if scheme.element.kind.value == "float_micro" else "int",
            scheme.element.exponent_bits, scheme.element.mantissa_bits, scheme.block_size,
            scheme.scale.exponent_bits)

    def layout(self, n):
        return _native.shard_layout(n, self.cs)

    def workspace(self, n, requant=False):
        return 16

    def _put(self, shard, c, values):
        so, eo, _ = self.layout(c)
        ss, es = O.compress(values, self.o)
        shard[so:so + len(ss)] = torch.from_numpy(np.frombuffer(ss, np.uint8).copy())
        shard[eo:eo + len(es)] = torch.from_numpy(np.frombuffer(es, np.uint8).copy())

    def _get(self, shard, c, n):
        so, eo, _ = self.layout(c)
        raw = shard.numpy().tobytes()
        return O.decompress(raw[so:], raw[eo:], n, self.o, np.float32)

    def quantize_into(self, x, shard, ws, flag):
        self._put(shard, x.numel(), x.double().numpy())

    def quantize_chunks(self, x, c, shards, stride, ws, flag):
        v = x.double().numpy()
        for j in range(-(-v.size // c)):
            self._put(shards[j * stride:(j + 1) * stride], c, v[j * c:(j + 1) * c])

    def dequant_sum(self, shards, rank_stride, nranks, n, c, chunk_stride, out, residual=None):
        acc = np.zeros(n, dtype=np.float32)
        for j in range(-(-n // c)):
            lo, hi = j * c, min(n, (j + 1) * c)
            for r in range(nranks):
                base = r * rank_stride + j * chunk_stride
                acc[lo:hi] += self._get(shards[base:], c, hi - lo)
        s = torch.from_numpy(acc).to(out.dtype)
        out.copy_(s if residual is None else residual.reshape(-1) + s)

    def requant(self, shards, rank_stride, nranks, n, c, out_shard, ws, flag):
        acc = np.zeros(n, dtype=np.float32)
        for r in range(nranks):
            acc += self._get(shards[r * rank_stride:], c, n)
        self._put(out_shard, c, acc.astype(np.float64))

    def reset_flag(self, flag):
        flag.fill_(-1)
