#!/bin/bash
# trips of the block-resident PCG kernel: parity tests that drive the direction solve, timings against the older
# persistent kernel (REGOT_B200_PCG_BLOCKS=0), then per-section cycle counts from an instrumented build
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_sparse_gpu.py tests/test_splr_gpu.py tests/test_step_api_gpu.py -x -q 2>&1 | tail -5 | tee gpurun_out/blocks_pytest.txt
timeout 200 python scripts/pcg_breakdown.py 3 2>&1 | tail -4 | tee gpurun_out/blocks_breakdown.txt
REGOT_B200_PCG_BLOCKS=0 timeout 200 python scripts/pcg_breakdown.py 3 2>&1 | tail -4 | tee -a gpurun_out/blocks_breakdown.txt
timeout 300 python scripts/solve_config.py B 2>&1 | grep -v "^   it" | tail -12 | tee gpurun_out/blocks_B.txt
make -C paper_2605_08793_b200/csrc clean > /dev/null
make -j16 -C paper_2605_08793_b200/csrc EXTRA=-DREGOT_PCG_TIMING > /dev/null 2>&1 || exit 1
REGOT_B200_PCG_FIXED_ITERS=1000 timeout 200 python scripts/pcg_breakdown.py 1 2>&1 | tail -3 | tee gpurun_out/blocks_timing.txt
