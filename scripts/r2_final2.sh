#!/bin/bash
# last state of round 2: smoke, GPU suite, both bench arms, launch list of one config-D solve, ncu --set full of the
# kernel-by-kernel PCG's kernels, configs A B C D E, preconditioner and panel-width tables
mkdir -p gpurun_out
export REGOT_B200_MAILBOX_TIMEOUT_S=300
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_full.txt 2>&1; tail -5 gpurun_out/pytest_gpu_full.txt | tee gpurun_out/pytest_gpu.txt
timeout 1200 python bench.py --gpus 1 --steps 5 --warmup 3 2>&1 | tail -1 > gpurun_out/bench.txt; cut -c1-300 gpurun_out/bench.txt
timeout 900 python bench.py --impl reference --gpus 1 --steps 2 --warmup 1 2>&1 | tail -1 > gpurun_out/bench_ref.txt; cut -c1-200 gpurun_out/bench_ref.txt
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 80000 --csv --log-file gpurun_out/r02_launches_D.csv \
    python scripts/solve_cloud.py D 0 > gpurun_out/r02_launches_D.log 2>&1
python scripts/launch_summary.py gpurun_out/r02_launches_D.csv gpurun_out/r02_launches_D_summary.csv | head -24
MAXIT=12 timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_spmv_panel|k_schur_w|k_schur_step|k_schur_diag|k_panel_combine|k_ell_values" -s 40 -c 12 \
    -o gpurun_out/r02_mk_D -f python scripts/solve_cloud.py D 0 > gpurun_out/r02_ncu_mk_D.log 2>&1; tail -1 gpurun_out/r02_ncu_mk_D.log
bash scripts/r2_e2e.sh > /dev/null 2>&1
REPS=2 timeout 900 python scripts/solve_cloud.py E 1 2>&1 | tail -10 > gpurun_out/e2e_E.txt
REPS=2 timeout 900 python scripts/solve_cloud.py D 0 2>&1 | tail -10 > gpurun_out/e2e_D.txt
bash scripts/r2_precond.sh > /dev/null 2>&1
{ WIDTHS="12800 10016 8352 7168" bash scripts/r2_ell_width.sh; echo "== pieces read from the CSR / CSC copy (REGOT_B200_PANEL_ELL=0)";
  REGOT_B200_PANEL_ELL=0 REPS=2 timeout 600 python scripts/solve_cloud.py D 0 2>&1 | grep -E "wall_s|spmv" | cut -c1-120; } > gpurun_out/r2_ell_width.txt 2>&1
ls gpurun_out | head -60
