#!/bin/bash
# Jacobi preconditioner of the Schur PCG: diag(S) (default) against D2 (REGOT_B200_SCHUR_DIAG=0) on configs A, B, C, D
mkdir -p gpurun_out
export REGOT_B200_MAILBOX_TIMEOUT_S=120
for SD in 1 0; do
  export REGOT_B200_SCHUR_DIAG=$SD
  for cfg in A B C; do
    echo "== schur_diag $SD config $cfg"; timeout 600 python scripts/solve_config.py $cfg 2>&1 | grep "\"rep\": 1" | cut -c1-330
  done
  echo "== schur_diag $SD config D"; REPS=2 timeout 600 python scripts/solve_cloud.py D 0 2>&1 | grep -E "wall_s|spmv" | cut -c1-330
done 2>&1 | tee gpurun_out/r2_precond.txt
