#!/bin/bash
# end-to-end checks after a direction-solve change: configs A, B, C solved to 1e-8, the paper's sizes against Sinkhorn
mkdir -p gpurun_out
export REGOT_B200_MAILBOX_TIMEOUT_S=120
for cfg in A B C; do
  echo "== config $cfg"; timeout 600 python scripts/solve_config.py $cfg 2>&1 | grep "rep\|launches" | grep -v "^   it"
done 2>&1 | tee gpurun_out/e2e_ABC.txt
timeout 900 python scripts/time_to_tol.py 2>&1 | tail -8 | tee gpurun_out/e2e_paper.txt
