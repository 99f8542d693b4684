#!/bin/bash
# correctness first, then timing, then (with NCU=1) one full ncu capture of the persistent PCG kernel
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_sparse_gpu.py tests/test_splr_gpu.py -m gpu -q -x 2>&1 | tail -5
timeout 300 python scripts/pcg_breakdown.py 3 2>&1 | tail -3
if [ -n "$NCU" ]; then
REGOT_B200_PCG_FIXED_ITERS=200 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pcg_schur -s 2 -c 1 \
    -o gpurun_out/pcg_prof -f python scripts/pcg_breakdown.py 3 > gpurun_out/ncu_pcg.log 2>&1
tail -3 gpurun_out/ncu_pcg.log
fi
