#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_full.txt 2>&1; tail -15 gpurun_out/pytest_gpu_full.txt | tee gpurun_out/pytest_gpu.txt
timeout 300 python scripts/time_sweeps.py 2>&1 | tee gpurun_out/time_sweeps.txt
timeout 300 python scripts/pcg_breakdown.py 3 2>&1 | tee gpurun_out/pcg_breakdown.txt
timeout 300 python scripts/pcg_breakdown.py 1 2>&1 | tee -a gpurun_out/pcg_breakdown.txt
