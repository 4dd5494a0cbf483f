"""A few eager launches of the comparison codecs at the 8B prefill shape
(for an ncu launch list: per-kernel times of the TopK / channel-INT stages)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_09510_b200 import baselines as bl  # noqa: E402

x = torch.randn(2048, 4096, device="cuda").to(torch.bfloat16)
for _ in range(2):
    bl.channelwise_int_compress_device(x, 4, check_finite=False)
    bl.topk_compress_device(x, bl.topk_budget(x.numel(), 2, 3.0), check_finite=False)
torch.cuda.synchronize()
