#!/bin/bash
# A/B of the GEMM variants (MXB200_GEMM_2CTA / _EPI / _STREAMK) on one B200.
# usage: gpurun -- 'bash scripts/gemm_ab.sh <tag> [ncu]'
tag=${1:-gemm_ab}
o=gpurun_out/$tag
mkdir -p $o
MXB200_GEMM_2CTA=1 timeout 400 python -m pytest tests/test_gpu_gemm.py -x -q > $o/tests_2cta.txt 2>&1
tail -3 $o/tests_2cta.txt
timeout 300 python scripts/gemm_bench.py --variants cublas,cublas+k1 > $o/ab_cublas.jsonl 2>&1
for two in 0 1; do for epi in 4 8; do
  MXB200_GEMM_2CTA=$two MXB200_GEMM_EPI=$epi timeout 300 python scripts/gemm_bench.py --variants ours_plain,ours_fused > $o/ab_2cta${two}_epi${epi}.jsonl 2>&1
done; done
if [ "$2" = ncu ]; then
for two in 0 1; do
MXB200_GEMM_2CTA=$two timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemm_mx -s 1 -c 1 -o $o/prof_gemm_2cta$two python scripts/gemm_bench.py --profile --filter "8b down_proj tp2" --variants ours_fused > $o/ncu_2cta$two.log 2>&1
python scripts/ncu_summary.py $o/prof_gemm_2cta$two.ncu-rep > $o/prof_gemm_2cta$two.summary.txt 2>&1
ncu -i $o/prof_gemm_2cta$two.ncu-rep --page raw --csv > $o/prof_gemm_2cta$two.raw.csv 2>&1
ncu -i $o/prof_gemm_2cta$two.ncu-rep --page details > $o/prof_gemm_2cta$two.details.txt 2>&1
rm -f $o/prof_gemm_2cta$two.ncu-rep
done
fi
for f in $o/ab_*.jsonl; do echo "== $f"; python -c "
import json,sys
for l in open('$f'):
    try: r=json.loads(l)
    except Exception: print(l.strip()[:300]); continue
    print(r['shape'], {k:v.get('us', v.get('error')) for k,v in r.items() if isinstance(v,dict)}, r.get('fused_shard_equals_k1_of_partial'))
"; done
