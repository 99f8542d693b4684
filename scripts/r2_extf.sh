#!/bin/bash
# extended-precision objective (default) against plain doubles (REGOT_B200_EXTENDED_F=0): time to 1e-8 and counts
mkdir -p gpurun_out
export REGOT_B200_MAILBOX_TIMEOUT_S=120
for ext in 1 0; do
  echo "=== REGOT_B200_EXTENDED_F=$ext"
  for cfg in A B C synth2:1600:1200:0.001 synth2:6400:4800:0.001 synth1-iid:3200:2400:0.001; do
    echo -n "$cfg: "; REGOT_B200_EXTENDED_F=$ext timeout 600 python scripts/solve_config.py $cfg 2>&1 | grep "\"rep\": 1" | cut -c1-330
  done
  echo -n "D: "; REGOT_B200_EXTENDED_F=$ext REPS=2 timeout 600 python scripts/solve_cloud.py D 0 2>&1 | grep "device_ms"
done 2>&1 | tee gpurun_out/extf.txt
