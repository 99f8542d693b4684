#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -5 | tee gpurun_out/pytest_gpu.txt
timeout 900 python bench.py --gpus 1 --steps 5 --warmup 3 2>&1 | tail -3 | tee gpurun_out/bench.txt
timeout 900 python bench.py --impl reference --gpus 1 --steps 2 --warmup 1 2>&1 | tail -2 | tee gpurun_out/bench_ref.txt
