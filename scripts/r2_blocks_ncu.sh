#!/bin/bash
# ncu --set full capture of the block-resident PCG kernel (200 fixed iterations on the config B pattern)
mkdir -p gpurun_out
REGOT_B200_PCG_FIXED_ITERS=200 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pcg_blocks -c 1 \
    -o gpurun_out/r2_blocks -f python scripts/pcg_breakdown.py 1 > gpurun_out/r2_blocks_ncu.log 2>&1
tail -3 gpurun_out/r2_blocks_ncu.log
