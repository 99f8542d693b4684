#!/bin/bash
# prefetch distance of the ELL stream (rows of 32 entries) at config D
for A in ${AHEADS:-0 256 512 1024 2048}; do
  echo "== ahead $A"
  REGOT_B200_PANEL_AHEAD=$A REPS=2 timeout 600 python scripts/solve_cloud.py D 0 2>&1 | grep -E "wall_s|spmv"
done
