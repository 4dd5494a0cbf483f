#!/bin/bash
# compute-sanitizer over the kernels with flags, spin-waits, PDL and
# same-kernel read-back (K4 k_fused_flow, K5 k_symm_flow, K5b k_symm2_flow)
# plus the K1/K2/K3 parity tests: memcheck (out-of-bounds / misaligned
# global and shared accesses), racecheck (shared-memory hazards), synccheck
# (illegal barrier use), initcheck (reads of uninitialised device memory).
# usage: gpurun --timeout 2400 -- 'bash scripts/sanitize.sh [tag]'
tag=${1:-san}
out=gpurun_out/$tag
mkdir -p $out
export MXB200_SYMM_TIMEOUT_MS=${MXB200_SYMM_TIMEOUT_MS:-20000}
SAN="compute-sanitizer --target-processes all --print-limit 50"
T_SYMM="tests/test_gpu_symm_multirank.py tests/test_gpu_symm.py"
run() {  # name tool tests...
  local name=$1 tool=$2
  shift 2
  timeout 900 $SAN --tool $tool python -m pytest -x -q -p no:cacheprovider "$@" \
    > $out/$name.log 2>&1
  echo "$name rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' $out/$name.log | tail -3 | tr '\n' ' ')" \
    | tee -a $out/summary.txt
}
run memcheck_symm memcheck $T_SYMM
run racecheck_symm racecheck $T_SYMM
run synccheck_symm synccheck $T_SYMM
run memcheck_flow memcheck tests/test_gpu_host.py::test_flow_kernel_nonfinite_flag tests/test_gpu_parity.py -k "fused or oneshot or twoshot or explicit or nonfinite or unit_counts or empty"
run racecheck_flow racecheck tests/test_gpu_host.py::test_flow_kernel_nonfinite_flag tests/test_gpu_parity.py -k "fused or oneshot or twoshot or explicit or nonfinite or unit_counts or empty"
run synccheck_flow synccheck tests/test_gpu_host.py::test_flow_kernel_nonfinite_flag tests/test_gpu_parity.py -k "fused or oneshot or twoshot or explicit or nonfinite or unit_counts or empty"
run initcheck_flow initcheck tests/test_gpu_host.py::test_flow_kernel_nonfinite_flag
# round 2: residual-fused stores, the device MXC1 kernel, E5M0 (packed k-bit
# scale) lean kernels -- K1/K2/K4 via the fused/two-shot parity cases
T_R2="tests/test_gpu_residual.py tests/test_gpu_mxc1.py"
run memcheck_r2 memcheck $T_R2 tests/test_gpu_parity.py -k "e5m0 or e4m0 or residual or serialize"
run racecheck_r2 racecheck $T_R2 tests/test_gpu_parity.py -k "e5m0 or e4m0"
run synccheck_r2 synccheck tests/test_gpu_parity.py -k "e5m0 or e4m0"
# the GEMM + all-gather push (peer stores from the epilogue, flag publish /
# acquire in the decode launch)
run memcheck_push memcheck tests/test_gpu_push.py
run racecheck_push racecheck tests/test_gpu_push.py
run synccheck_push synccheck tests/test_gpu_push.py
cat $out/summary.txt
