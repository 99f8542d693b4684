#!/bin/bash
# state at the end of round 2 (after the CSC-ordered values and the guessed count sweep): smoke, GPU suite, both bench
# arms, launch list of one config-D solve, configs A-E end to end
mkdir -p gpurun_out
export REGOT_B200_MAILBOX_TIMEOUT_S=300
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_full.txt 2>&1; tail -5 gpurun_out/pytest_gpu_full.txt | tee gpurun_out/pytest_gpu.txt
timeout 1200 python bench.py --gpus 1 --steps 5 --warmup 3 2>&1 | tail -1 > gpurun_out/bench.txt; cut -c1-300 gpurun_out/bench.txt
timeout 900 python bench.py --impl reference --gpus 1 --steps 2 --warmup 1 2>&1 | tail -1 > gpurun_out/bench_ref.txt; cut -c1-200 gpurun_out/bench_ref.txt
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 80000 --csv --log-file gpurun_out/r02c_launches_D.csv \
    python scripts/solve_cloud.py D 0 > gpurun_out/r02c_launches_D.log 2>&1
python scripts/launch_summary.py gpurun_out/r02c_launches_D.csv gpurun_out/r02c_launches_D_summary.csv | head -24
bash scripts/r2_e2e.sh > /dev/null 2>&1
ls gpurun_out | head -60
