"""Back-to-back cost of the NVLink kernels (K5 one-shot, K5b two-shot) at
world size 1: 50 calls captured in one CUDA graph, replayed, CUDA-event
timed.  World 1 still runs the whole kernel (quantise, flag publish/acquire,
pull, dequant-sum) over the one local shard.  The switches compared:
MXB200_PDL (programmatic dependent launch) and MXB200_SYMM_FENCE (extra
fence.sc.sys around the flags).

    MXB200_PDL=0 MXB200_SYMM_FENCE=1 MXB200_SYMM_CTAS=296 python scripts/symm_bench.py [n]
"""

import json
import os
import socket
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2411_09510_b200.collective import SymmetricAllReduce  # noqa: E402


def main():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(s.getsockname()[1])
    s.close()
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048 * 4096
    calls, reps = 50, 40
    x = torch.randn(n, device="cuda").to(torch.bfloat16)
    for algo in ("oneshot", "twoshot"):
        car = SymmetricAllReduce("fp4_e2m1:32:e8m0", n, algo=algo)
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            for _ in range(3):
                car(x)
            st.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                for _ in range(calls):
                    car(x)
            for _ in range(3):
                g.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            st.synchronize()
            e0.record(st)
            for _ in range(reps):
                g.replay()
            e1.record(st)
            e1.synchronize()
        car.check_status()
        print(json.dumps({"algo": algo, "pdl": os.environ.get("MXB200_PDL", "1"),
                          "fence": os.environ.get("MXB200_SYMM_FENCE", "0"),
                          "ctas_cap": os.environ.get("MXB200_SYMM_CTAS", "592"), "n": n,
                          "us_per_call": round(e0.elapsed_time(e1) * 1e3 / (calls * reps), 3)}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
