#!/bin/bash
# ncu evidence for profiles/: (1) launch list of a bench run, (2) full captures of the K1 sweep (resident and
# on-the-fly cost), the LSE sweeps, the persistent PCG kernel and the half mat-vec of the kernel-by-kernel PCG.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
    --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gradient_sweep -s 3 -c 2 \
    -o gpurun_out/k1_prof -f python scripts/time_gradient.py 10000 10000 8 > gpurun_out/ncu_k1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_row_lse_sweep|k_col_lse_sweep" -s 2 -c 2 \
    -o gpurun_out/lse_prof -f python scripts/solve_config.py B > gpurun_out/ncu_lse.log 2>&1
REGOT_B200_PCG_FIXED_ITERS=200 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pcg_schur -s 2 -c 1 \
    -o gpurun_out/pcg_prof -f python scripts/pcg_breakdown.py 1 > gpurun_out/ncu_pcg.log 2>&1
MAXIT=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gradient_sweep -s 2 -c 1 \
    -o gpurun_out/k1_cloud_prof -f python scripts/solve_cloud.py E 1 10000 > gpurun_out/ncu_k1cloud.log 2>&1
MAXIT=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv -s 40 -c 2 \
    -o gpurun_out/spmv_D_prof -f python scripts/solve_cloud.py D 0 > gpurun_out/ncu_spmvD.log 2>&1
ls -la gpurun_out/ | tail -14
