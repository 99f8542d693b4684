#!/bin/bash
# compute-sanitizer memcheck + initcheck over the kernel-by-kernel PCG (ELL stream plan and kernel, Schur diagonal) and the
# sharded loopback tests; clusters off (memcheck reports the block-resident kernel's self-addressed shared::cluster bulk
# copies as "not located in remote CTA")
mkdir -p gpurun_out
export REGOT_B200_PCG_BLOCKS_CLUSTER=0
for tool in memcheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest tests/test_sparse_gpu.py tests/test_sharded_loopback_gpu.py "tests/test_pcg_blocks_gpu.py::test_schur_diagonal_preconditioner_against_d2_on_clustered_clouds" -m gpu -q -x > gpurun_out/r2_sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/r2_sanitize_$tool.log | tail -3
done
