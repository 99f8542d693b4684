#!/bin/bash
# ncu capture of the K1 sweep kernel at config-B size.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gradient_sweep -s 3 -c 2 \
    -o gpurun_out/k1_prof -f python scripts/time_gradient.py 10000 10000 8 > gpurun_out/ncu_k1.log 2>&1
tail -5 gpurun_out/ncu_k1.log
ls -la gpurun_out/
