#!/bin/bash
# config D on one GPU: launch list of a short solve (MAXIT iterations) + `ncu --set full` captures of the panel
# mat-vec (both halves), K1, K7, K8 and the top-k sweeps
mkdir -p gpurun_out
MAXIT=11 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv \
    --log-file gpurun_out/r2_launches_D.csv python scripts/solve_cloud.py D 0 > gpurun_out/r2_launches_D.log 2>&1
tail -12 gpurun_out/r2_launches_D.log
python scripts/launch_summary.py gpurun_out/r2_launches_D.csv > gpurun_out/r2_launches_D_summary.csv 2>&1; head -30 gpurun_out/r2_launches_D_summary.csv
MAXIT=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv_panel -s 20 -c 2 \
    -o gpurun_out/r2_panel -f python scripts/solve_cloud.py D 0 > gpurun_out/r2_ncu_panel.log 2>&1
tail -3 gpurun_out/r2_ncu_panel.log
MAXIT=1 timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_gradient_sweep|k_row_lse_sweep|k_col_lse_sweep|k_topk_sweep" -s 6 -c 12 \
    -o gpurun_out/r2_sweeps_D -f python scripts/solve_cloud.py D 0 > gpurun_out/r2_ncu_sweeps.log 2>&1
tail -3 gpurun_out/r2_ncu_sweeps.log
