#!/bin/bash
# block-resident PCG on small and mid-size patterns (single cluster / block rows as clusters / through L2 / old kernel)
mkdir -p gpurun_out
export REGOT_B200_MAILBOX_TIMEOUT_S=20
for mode in ${MODES:-"X=1" "REGOT_B200_PCG_BLOCKS_CLUSTER=0" "REGOT_B200_PCG_BLOCKS=0"}; do
  for cfg in ${CFGS:-A synth1-iid:1600:1200:0.001 synth1-iid:6400:4800:0.001}; do
    echo "== $mode $cfg"
    env $mode REGOT_B200_PCG_BLOCKS_INFO=1 timeout 120 python scripts/solve_config.py $cfg 2>&1 | grep "rep\|pcg \|rror" | sort | uniq -c | sort -rn | head -6
  done
done 2>&1 | tee gpurun_out/blocks_small.txt
