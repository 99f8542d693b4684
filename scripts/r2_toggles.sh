#!/bin/bash
# optional faster variants of the Sinkhorn candidate chain, now that the objective is extended: tests and times
mkdir -p gpurun_out
export REGOT_B200_MAILBOX_TIMEOUT_S=120
for tg in "X=1" "REGOT_B200_LSE_FAST_SHIFT=1" "REGOT_B200_FAST_CHAIN=1"; do
  echo "=== $tg"
  env $tg timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3
  for cfg in A B C synth2:1600:1200:0.001; do
    echo -n "$cfg: "; env $tg timeout 600 python scripts/solve_config.py $cfg 2>&1 | grep "\"rep\": 1" | cut -c1-200
  done
  echo -n "D: "; env $tg REPS=2 timeout 600 python scripts/solve_cloud.py D 0 2>&1 | grep "device_ms" | cut -c1-200
done 2>&1 | tee gpurun_out/toggles.txt
