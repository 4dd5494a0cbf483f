"""Debug: world-1 SymmetricAllReduce vs CompressedAllReduce on the 8B shape."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1")
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
from paper_2411_09510_b200.collective import CompressedAllReduce, SymmetricAllReduce
from paper_2411_09510_b200.formats import parse_scheme
from paper_2411_09510_b200.synth import rank_partials
from oracle import mx_oracle as O
spec = "fp4_e2m1:32:e8m0"
sch = parse_scheme(spec)
shape = (2048, 4096); n = shape[0] * shape[1]
host = rank_partials(shape, 1, seed=0)[0]
x = torch.from_numpy(host).to("cuda", torch.bfloat16)
ref = O.allreduce_oneshot([x.float().cpu().numpy().astype(np.float64).ravel()], O.scheme(spec))
want = torch.from_numpy(np.asarray(ref, np.float32)).to(torch.bfloat16)
car = CompressedAllReduce(sch, n, algo="oneshot", out_dtype=torch.bfloat16)
a = car(x).clone().cpu()
print("car vs oracle", torch.equal(a.view(torch.int16), want.view(torch.int16)))
for algo in ("oneshot", "twoshot"):
    sar = SymmetricAllReduce(sch, n, out_dtype=torch.bfloat16, algo=algo)
    for k in range(3):
        b = sar(x).clone(); torch.cuda.synchronize(); sar.check_status()
        b = b.reshape(-1).cpu()
        d = (b.view(torch.int16) != want.view(torch.int16))
        print(algo, k, "sar vs oracle", not bool(d.any()), int(d.sum()), "first", d.nonzero()[:5].ravel().tolist())
        if d.any():
            i = d.nonzero()[0].item()
            print("  got", b[i-2:i+3].tolist(), "want", want[i-2:i+3].tolist())
dist.destroy_process_group()
