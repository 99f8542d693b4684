#!/bin/bash
# after a kernel change: whole GPU suite, then configs A, B, D with the time split
mkdir -p gpurun_out
export REGOT_B200_MAILBOX_TIMEOUT_S=120
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -8 | tee gpurun_out/pytest_gpu.txt
for cfg in A B; do
  echo "== config $cfg"; timeout 600 python scripts/solve_config.py $cfg 2>&1 | grep "\"rep\": 1\|launches" | grep -v "^   it"
done 2>&1 | tee gpurun_out/check_AB.txt
REPS=2 timeout 600 python scripts/solve_cloud.py D 0 2>&1 | tail -12 | tee gpurun_out/check_D.txt
