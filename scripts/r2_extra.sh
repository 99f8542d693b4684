bash scripts/r2_precond.sh > /dev/null 2>&1
{ WIDTHS="12800 10016 8352 7168" bash scripts/r2_ell_width.sh; echo "== pieces read from the CSR / CSC copy (REGOT_B200_PANEL_ELL=0)";
  REGOT_B200_PANEL_ELL=0 REPS=2 timeout 600 python scripts/solve_cloud.py D 0 2>&1 | grep -E "wall_s|spmv" | cut -c1-120; } > gpurun_out/r2_ell_width.txt 2>&1
MAXIT=12 timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_schur_diag|k_ell_values|k_panel_combine" -s 3 -c 4 \
    -o gpurun_out/r02_diag_D -f python scripts/solve_cloud.py D 0 > gpurun_out/r02_ncu_diag_D.log 2>&1; tail -1 gpurun_out/r02_ncu_diag_D.log
