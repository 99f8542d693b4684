#!/bin/bash
# The numbers recorded under profiles/: both bench arms, then every BASELINE config solved on one GPU.
mkdir -p gpurun_out
timeout 900 python bench.py --gpus 1 --steps 5 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_line.json
timeout 900 python bench.py --impl reference --gpus 1 --steps 2 --warmup 1 2>&1 | tail -1 > gpurun_out/bench_reference_line.json
(timeout 600 python scripts/solve_config.py A 2>&1 | grep -v "^   it") > gpurun_out/solve_A.txt
(timeout 900 python scripts/solve_config.py C 2>&1 | grep -v "^   it") > gpurun_out/solve_C.txt
REPS=2 timeout 900 python scripts/solve_cloud.py D 0 > gpurun_out/cloud_D.txt 2>&1
timeout 900 python scripts/solve_cloud.py E 1 > gpurun_out/cloud_E.txt 2>&1
timeout 300 python scripts/time_sweeps.py > gpurun_out/time_sweeps.txt 2>&1
cut -c1-300 gpurun_out/bench_line.json; echo; tail -n 4 gpurun_out/solve_A.txt gpurun_out/solve_C.txt | cut -c1-300
