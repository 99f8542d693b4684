#!/bin/bash
# panel width x prefetch distance of the ELL stream at config D
for W in ${WIDTHS:-12800 10016 8352}; do
 for A in ${AHEADS:-0 256 512 1024}; do
  echo "== width $W ahead $A"
  REGOT_B200_PANEL_WIDTH=$W REGOT_B200_PANEL_AHEAD=$A REPS=2 timeout 600 python scripts/solve_cloud.py D 0 2>&1 | grep -E "wall_s|spmv" | cut -c1-100
 done
done
