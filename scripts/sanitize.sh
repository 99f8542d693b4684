#!/bin/bash
# compute-sanitizer passes over the GPU tests (memcheck: out-of-bounds / misaligned; racecheck: shared-memory
# hazards; synccheck: barrier misuse).  The full-size property tests are left out (too slow under the tools).
mkdir -p gpurun_out
T="tests --ignore=tests/test_fullsize_gpu.py"
for tool in memcheck racecheck synccheck; do
  timeout 2400 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest $T -m gpu -q -x > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/sanitize_$tool.log | tail -3
done
