#!/bin/bash
# us per CG iteration (1000 fixed iterations) of the direction-solve kernels at several sizes
mkdir -p gpurun_out
export REGOT_B200_MAILBOX_TIMEOUT_S=30
for prob in synth1-iid:1000:1000:0.01 synth1-iid:1600:1200:0.001 synth1-iid:3200:2400:0.001 synth1-iid:6400:4800:0.001 synth2:20000:5000:0.0005 ""; do
  for mode in "X=1" "REGOT_B200_PCG_BLOCKS_CLUSTER=0" "REGOT_B200_PCG_BLOCKS=0" ${EXTRA_MODES}; do
    echo "== ${prob:-config B} | $mode"
    env $mode PROBLEM=$prob REGOT_B200_PCG_BLOCKS_INFO=1 timeout 120 python scripts/pcg_breakdown.py 1 2>&1 | grep "fixed=1000\|pcg blocks: [0-9]" | sort | uniq | tail -2
  done
done 2>&1 | tee gpurun_out/blocks_iter.txt
