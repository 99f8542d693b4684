#!/bin/bash
# pattern reuse (regot_b200_set_pattern_reuse / REGOT_B200_PATTERN_DRIFT): new tests, then configs D, B, C with the
# reference's fixed rule against drift tolerances 0.05 / 0.2 / 0.5
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke.txt
export REGOT_B200_MAILBOX_TIMEOUT_S=300
timeout 900 python -m pytest tests/test_pattern_reuse_gpu.py tests/test_sharded_loopback_gpu.py -m gpu -q -s -k "reuse or pattern" 2>&1 | tail -25 | tee gpurun_out/pytest_reuse.txt
{
for tol in 0 0.05 0.2 0.5; do
  echo "== config D, REGOT_B200_PATTERN_DRIFT=$tol"
  REGOT_B200_PATTERN_DRIFT=$tol REPS=2 timeout 600 python scripts/solve_cloud.py D 0 2>&1 | grep -E "wall_s|topk"
done
for cfg in B C; do for tol in 0 0.05 0.2 0.5; do
  echo "== config $cfg, REGOT_B200_PATTERN_DRIFT=$tol"
  REGOT_B200_PATTERN_DRIFT=$tol timeout 600 python scripts/solve_config.py $cfg 2>&1 | grep "rep\|launches" | grep -v "^   it"
done; done
} 2>&1 | tee gpurun_out/r02c_pattern_reuse.txt
