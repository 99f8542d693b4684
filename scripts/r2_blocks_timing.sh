#!/bin/bash
# per-section cycle counts of the block-resident PCG kernel (instrumented build, on the box only)
mkdir -p gpurun_out
make -C paper_2605_08793_b200/csrc clean > /dev/null
make -j16 -C paper_2605_08793_b200/csrc EXTRA=-DREGOT_PCG_TIMING > /dev/null 2>&1 || exit 1
export REGOT_B200_PCG_FIXED_ITERS=${FIXED:-1000}
for prob in ${PROBS:-synth1-iid:1600:1200:0.001 synth1-iid:6400:4800:0.001 B}; do
  for mode in "X=1" "REGOT_B200_PCG_BLOCKS_CLUSTER=0"; do
    echo "== $prob | $mode"
    if [ "$prob" = B ]; then pp=""; else pp=$prob; fi
    env $mode PROBLEM=$pp timeout 200 python scripts/pcg_breakdown.py 1 2>&1 | grep "kcycles\|fixed=" | tail -2
  done
done 2>&1 | tee gpurun_out/blocks_timing.txt
