"""Where the reference-API round trip spends its time (host arrays in and
out): compress_tensor(np.float32 [2048x4096]) -> CompressedTensor ->
decompress_tensor(ct, np.float32), each step timed separately (ms)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2411_09510_b200 import codec  # noqa: E402
from paper_2411_09510_b200.formats import parse_scheme  # noqa: E402
from paper_2411_09510_b200.synth import rank_partials  # noqa: E402


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return round(1e3 * sorted(ts)[len(ts) // 2], 3), r


def main():
    sch = parse_scheme("fp4_e2m1:32:e8m0")
    x = rank_partials((2048, 4096), 1, seed=0)[0].astype(np.float32)
    res = {}
    res["to_device_values"], (xd, shape) = t(lambda: codec._to_device_values(x))
    res["compress_device_checked"], dct = t(lambda: codec.compress_tensor_device(xd, sch))
    res["compress_device_nocheck"], _ = t(lambda: codec.compress_tensor_device(xd, sch, False))
    res["to_host"], ct = t(lambda: dct.to_host())
    res["compress_tensor_total"], ct = t(lambda: codec.compress_tensor(x, sch))
    res["upload"], up = t(lambda: codec._upload(ct))
    res["decompress_device"], dd = t(lambda: codec.decompress_tensor_device(up, torch.float32))
    res["d2h_numpy"], _ = t(lambda: dd.cpu().numpy())
    res["decompress_tensor_total"], _ = t(lambda: codec.decompress_tensor(ct, np.float32))
    res["np_alloc_32MB_touch"], _ = t(lambda: np.ones(x.size, np.float32))
    res["np_add_inplace"], _ = t(lambda: np.add(x, x, out=np.empty_like(x)))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
