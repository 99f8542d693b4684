#!/bin/bash
# quick trip: GPU tests (stop at first failure), PCG timing, short bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_full.txt 2>&1; tail -25 gpurun_out/pytest_gpu_full.txt | tee gpurun_out/pytest_gpu.txt
timeout 300 python scripts/pcg_breakdown.py 3 2>&1 | tail -5 | tee gpurun_out/pcg_breakdown.txt
timeout 900 python bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu 2>&1 | tail -3 | tee gpurun_out/bench_quick.txt
