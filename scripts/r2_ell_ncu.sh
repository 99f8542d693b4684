#!/bin/bash
# `ncu --set full` capture of the ELL-stream panel mat-vec (both halves) at config D; short solve
mkdir -p gpurun_out
MAXIT=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv_panel -s 20 -c 2 \
    -o gpurun_out/r2_panel_ell -f python scripts/solve_cloud.py D 0 > gpurun_out/r2_ncu_panel_ell.log 2>&1
tail -3 gpurun_out/r2_ncu_panel_ell.log
