#!/bin/bash
# per-section cycle counts of the block-resident PCG kernel (instrumented build, on the box only)
mkdir -p gpurun_out
make -C paper_2605_08793_b200/csrc clean > /dev/null
make -j16 -C paper_2605_08793_b200/csrc EXTRA=-DREGOT_PCG_TIMING > /dev/null 2>&1 || exit 1
REGOT_B200_PCG_FIXED_ITERS=${FIXED:-200} timeout 200 python scripts/pcg_breakdown.py 1 2>&1 | tail -12 | tee gpurun_out/blocks_timing.txt
