#!/bin/bash
# panel width of the panel mat-vec at config D: narrower panels leave more of the SM's 256 KB to L1, which is where the
# in-flight lines of the matrix stream land
for W in ${WIDTHS:-12800 10016 8352 7168 6272 5568}; do
  echo "== width $W"
  REGOT_B200_PANEL_WIDTH=$W REPS=2 timeout 600 python scripts/solve_cloud.py D 0 2>&1 | grep -E "wall_s|spmv" | cut -c1-120
done
