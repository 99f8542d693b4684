#!/bin/bash
# the candidate chain with the gradient-sweep form of the Sinkhorn update (REGOT_B200_FAST_CHAIN=1): tests + times
mkdir -p gpurun_out
export REGOT_B200_MAILBOX_TIMEOUT_S=120
for fc in 0 1; do
  echo "== FAST_CHAIN=$fc"
  for cfg in A B; do
    REGOT_B200_FAST_CHAIN=$fc timeout 300 python scripts/solve_config.py $cfg 2>&1 | grep "\"rep\": 1\|row_lse\|col_lse\|gradient "
  done
  REGOT_B200_FAST_CHAIN=$fc REPS=2 timeout 600 python scripts/solve_cloud.py D 0 2>&1 | grep "device_ms\|row_lse\|col_lse\|gradient "
done 2>&1 | tee gpurun_out/fastchain.txt
REGOT_B200_FAST_CHAIN=1 timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -12 | tee gpurun_out/fastchain_pytest.txt
