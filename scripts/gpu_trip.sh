#!/bin/bash
# GPU trip: parity tests, K1 timing.  Output under gpurun_out/.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 | tee gpurun_out/pytest_gpu.txt
timeout 300 python scripts/time_gradient.py 10000 10000 20 2>&1 | tee gpurun_out/time_gradient.txt
