#!/bin/bash
# Round-2 profiling pass (one gpurun call): ncu launch list of the default
# bench, --set full captures of K4 / K1-lean / K2-lean, and the range-replay
# DRAM traffic (reads AND write-backs) of each over 16 back-to-back launches.
# usage: gpurun --timeout 1500 -- 'bash scripts/gpu_profile_r02.sh [tag]'
tag=${1:-prof}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/smi.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $out/launches.csv python bench.py --profile > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_fused_flow -s 1 -c 1 \
  -o $out/prof_kfused python scripts/range_traffic.py --kernel k4 --sets 4 > $out/ncu0.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_quant_lean -s 1 -c 1 \
  -o $out/prof_kquant python scripts/range_traffic.py --kernel k1 --sets 4 > $out/ncu1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_dqsum_lean -s 1 -c 1 \
  -o $out/prof_kdqsum python scripts/range_traffic.py --kernel k2 --sets 4 > $out/ncu2.log 2>&1
for k in k4 k1 k2; do
  for shp in 2048,4096 4096,8192; do
    s=16; [ $shp = 4096,8192 ] && s=8
    timeout 300 ncu --replay-mode range --clock-control none --csv \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --log-file $out/range_${k}_${shp/,/x}.csv python scripts/range_traffic.py --kernel $k \
      --shape $shp --sets $s > $out/range_${k}_${shp/,/x}.log 2>&1
  done
done
for r in prof_kfused prof_kquant prof_kdqsum; do
  if [ -f $out/$r.ncu-rep ]; then
    python scripts/ncu_summary.py $out/$r.ncu-rep > $out/$r.summary.txt 2>&1
    ncu -i $out/$r.ncu-rep --page details > $out/$r.details.txt 2>&1
    ncu -i $out/$r.ncu-rep --page raw --csv > $out/$r.raw.csv 2>&1
    [ "${KEEP_REP:-0}" = 1 ] || rm -f $out/$r.ncu-rep
  fi
done
cat $out/prof_*.summary.txt; tail -4 $out/range_*.csv
du -sh $out
