#!/bin/bash
# trips of the block-resident PCG kernel: parity tests that drive the direction solve, timings of its forms (block
# rows as clusters / everything through L2) against the older persistent kernel, per-section cycle counts
mkdir -p gpurun_out
REGOT_B200_PCG_BLOCKS_INFO=1 timeout 200 python scripts/pcg_breakdown.py 3 2>&1 | tail -6 | tee gpurun_out/blocks_breakdown.txt
REGOT_B200_PCG_BLOCKS_CLUSTER=0 timeout 200 python scripts/pcg_breakdown.py 3 2>&1 | tail -2 | tee -a gpurun_out/blocks_breakdown.txt
REGOT_B200_PCG_BLOCKS_INFO=1 timeout 100 python scripts/solve_config.py A 2>&1 | grep "rep\|pcg \|rror" | sort | uniq -c | tee gpurun_out/blocks_A.txt
timeout 600 python -m pytest tests/test_sparse_gpu.py tests/test_splr_gpu.py tests/test_step_api_gpu.py -x -q --timeout 120 2>&1 | tail -8 | tee gpurun_out/blocks_pytest.txt
timeout 300 python scripts/solve_config.py B 2>&1 | grep "rep\|pcg " | tee gpurun_out/blocks_B.txt
if [ -n "$PAPER" ]; then timeout 600 python scripts/time_to_tol.py 2>&1 | tail -8 | tee gpurun_out/blocks_paper.txt; fi
if [ -n "$TIMING" ]; then
make -C paper_2605_08793_b200/csrc clean > /dev/null
make -j16 -C paper_2605_08793_b200/csrc EXTRA=-DREGOT_PCG_TIMING > /dev/null 2>&1 || exit 1
REGOT_B200_PCG_FIXED_ITERS=1000 timeout 200 python scripts/pcg_breakdown.py 1 2>&1 | tail -3 | tee gpurun_out/blocks_timing.txt
fi
