out=gpurun_out/${SAN_OUT:-san_push3}; mkdir -p $out
export MXB200_SYMM_TIMEOUT_MS=20000
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --target-processes all --print-limit 50 --tool $tool python -m pytest -x -q -p no:cacheprovider tests/test_gpu_push.py ${PUSH_K:+-k "$PUSH_K"} > $out/$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' $out/$tool.log | tail -3 | tr '\n' ' ')" | tee -a $out/summary.txt
done
