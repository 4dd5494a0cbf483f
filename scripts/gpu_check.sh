#!/bin/bash
# One gpurun call: GPU tests, bench, membench, ncu launch list and full
# captures of the fused kernel and of K1/K2 (unfused run).
# usage: gpurun --timeout 1500 -- 'bash scripts/gpu_check.sh [tag] [tests|notests]'
tag=${1:-dev}
mode=${2:-tests}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/smi.txt 2>&1
if [ "$mode" = tests ]; then
  timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15 > $out/tests.txt
fi
timeout 300 python bench.py > $out/bench.json 2> $out/bench.err
timeout 120 python scripts/membench.py > $out/membench.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/launches.csv python bench.py --profile > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none -k regex:k_fused -s 1 -c 1 \
  -o $out/prof_kfused python bench.py --profile > $out/ncu0.log 2>&1
MXB200_FUSED=0 timeout 300 ncu --set full --clock-control none -k regex:k_quant -s 2 -c 1 \
  -o $out/prof_kquant python bench.py --profile > $out/ncu1.log 2>&1
MXB200_FUSED=0 timeout 300 ncu --set full --clock-control none -k regex:k_dqsum -s 1 -c 1 \
  -o $out/prof_kdqsum python bench.py --profile > $out/ncu2.log 2>&1
cat $out/tests.txt 2>/dev/null | tail -3
cat $out/bench.json
tail -3 $out/bench.err
cat $out/membench.json
# reports are large: summarise on the box, bring back text only
for r in prof_kfused prof_kquant prof_kdqsum; do
  if [ -f $out/$r.ncu-rep ]; then
    python scripts/ncu_summary.py $out/$r.ncu-rep > $out/$r.summary.txt 2>&1
    ncu -i $out/$r.ncu-rep --page details > $out/$r.details.txt 2>&1
    ncu -i $out/$r.ncu-rep --page source --csv --print-source sass > $out/$r.sass.csv 2>&1
    ncu -i $out/$r.ncu-rep --page raw --csv > $out/$r.raw.csv 2>&1
    [ "${KEEP_REP:-0}" = 1 ] || rm -f $out/$r.ncu-rep
  fi
done
du -sh $out
