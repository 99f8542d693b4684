#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_full.txt 2>&1; tail -15 gpurun_out/pytest_gpu_full.txt | tee gpurun_out/pytest_gpu.txt
timeout 300 python scripts/time_sweeps.py 2>&1 | tee gpurun_out/time_sweeps.txt
timeout 300 python scripts/time_gradient.py 10000 10000 20 2>&1 | tee gpurun_out/time_gradient.txt
timeout 900 python bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu 2>&1 | tail -3 | tee gpurun_out/bench_quick.txt
