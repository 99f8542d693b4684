#!/bin/bash
# ncu evidence for profiles/: (1) launch list of a short bench run, (2) full capture of the K1 sweep,
# (3) full capture of the LSE sweeps and one persistent PCG solve.
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gradient_sweep -s 3 -c 2 \
    -o gpurun_out/k1_prof -f python scripts/time_gradient.py 10000 10000 8 > gpurun_out/ncu_k1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_row_lse_sweep|k_col_lse_sweep" -s 2 -c 2 \
    -o gpurun_out/lse_prof -f python scripts/solve_config.py B > gpurun_out/ncu_lse.log 2>&1
ls -la gpurun_out/ | tail -12
