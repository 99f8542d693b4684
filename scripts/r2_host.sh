#!/bin/bash
# where the host-side time of an SPLR iteration goes (REGOT_B200_STEP_TIMING=1), overlap on/off
export REGOT_B200_MAILBOX_TIMEOUT_S=120
for cfg in synth2:1600:1200:0.001 B; do
  echo "== $cfg"
  REGOT_B200_STEP_TIMING=1 timeout 300 python scripts/solve_config.py $cfg 2>&1 | grep "rep\": 1\|run_splr sections" | tail -6
  echo "-- overlap=1"
  timeout 300 python scripts/solve_config.py $cfg 1 2>&1 | grep "rep\": 1"
done 2>&1 | tee gpurun_out/host_timing.txt
