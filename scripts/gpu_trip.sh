#!/bin/bash
# One GPU round trip: smoke, GPU parity tests, both bench arms.  Outputs land in gpurun_out/.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -3 gpurun_out/smoke.txt
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_full.txt 2>&1; tail -40 gpurun_out/pytest_gpu_full.txt | tee gpurun_out/pytest_gpu.txt
timeout 900 python bench.py --gpus 1 --steps 5 --warmup 3 2>&1 | tail -3 | tee gpurun_out/bench.txt
timeout 900 python bench.py --impl reference --gpus 1 --steps 2 --warmup 1 2>&1 | tail -2 | tee gpurun_out/bench_ref.txt
