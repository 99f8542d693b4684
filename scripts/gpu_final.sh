#!/bin/bash
# Evidence for the last state of the round: sanitizer passes over the tests that drive the PCG kernels, the launch list
# of a bench run, a full capture of the persistent PCG kernel, and the other BASELINE configs.
mkdir -p gpurun_out
for tool in memcheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest tests/test_sparse_gpu.py tests/test_splr_gpu.py tests/test_bench_protocol_gpu.py -m gpu -q -x > gpurun_out/sanitize_c_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitize_c_$tool.log | tail -2
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
    --log-file gpurun_out/launches_bench_c.csv python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/bench_under_ncu_c.log 2>&1
REGOT_B200_PCG_FIXED_ITERS=200 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pcg_schur -s 2 -c 1 \
    -o gpurun_out/pcg_prof_c -f python scripts/pcg_breakdown.py 1 > gpurun_out/ncu_pcg_c.log 2>&1
bash scripts/gpu_record.sh
