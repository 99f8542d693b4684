#!/bin/bash
# one `ncu --set full` capture of the panel mat-vec (both halves) and of K1 at config D; short solve (MAXIT iterations)
mkdir -p gpurun_out
MAXIT=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv_panel -s 20 -c 2 \
    -o gpurun_out/r2_panel -f python scripts/solve_cloud.py D 0 > gpurun_out/r2_ncu_panel.log 2>&1
tail -3 gpurun_out/r2_ncu_panel.log
MAXIT=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gradient_sweep -s 6 -c 1 \
    -o gpurun_out/r2_k1_D -f python scripts/solve_cloud.py D 0 > gpurun_out/r2_ncu_k1.log 2>&1
tail -3 gpurun_out/r2_ncu_k1.log
