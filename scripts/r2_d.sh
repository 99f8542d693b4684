#!/bin/bash
# config D on one GPU: solve + where the time goes (scripts/solve_cloud.py), old vs panel mat-vec
set -x
REPS=2 python scripts/solve_cloud.py D 0 2>&1 | tail -12
REGOT_B200_PANEL_SPMV=0 REPS=2 python scripts/solve_cloud.py D 0 2>&1 | tail -10
