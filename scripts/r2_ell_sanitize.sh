#!/bin/bash
# compute-sanitizer over the kernel-by-kernel PCG with the panel mat-vec (ELL stream): memcheck, initcheck
# (uninitialised device reads), racecheck, synccheck
mkdir -p gpurun_out
T="tests/test_sparse_gpu.py -k panel"
for tool in memcheck initcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest $T -m gpu -q -x > gpurun_out/ell_sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/ell_sanitize_$tool.log | tail -3
done
grep -E "Uninitialized|at .*\(|in .*k_" gpurun_out/ell_sanitize_initcheck.log | sort | uniq -c | sort -rn | head -30
