#!/bin/bash
# Round-2 confirmation pass (one gpurun call): GPU tests, smoke, the default
# bench line, the bench under --force-dist (world-1 NCCL: the TP=N code
# path), then the profiling pass (launch list, --set full captures, range
# traffic).  usage: gpurun --timeout 2400 -- 'bash scripts/gpu_final_r02.sh [tag]'
tag=${1:-final}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > $out/tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1
timeout 600 python bench.py > $out/bench.json 2> $out/bench.err
timeout 600 python bench.py --force-dist --steps 200 --warmup 5 --no-70b > $out/bench_dist.json 2> $out/bench_dist.err
bash scripts/gpu_profile_r02.sh $tag/prof > $out/profile.log 2>&1
cat $out/tests.txt $out/smoke.txt
tail -c 600 $out/bench.json
