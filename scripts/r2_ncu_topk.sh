#!/bin/bash
# ncu --set full of the three top-k sweeps at config D (first refresh of a solve: histogram, count, write)
mkdir -p gpurun_out
MAXIT=1 timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_topk_sweep|k_compact" -c 4 \
    -o gpurun_out/r02c_topk_D -f python scripts/solve_cloud.py D 0 > gpurun_out/r02c_ncu_topk.log 2>&1
tail -3 gpurun_out/r02c_ncu_topk.log
python scripts/ncu_extract.py gpurun_out/r02c_ncu_topk_D.json topk_D=gpurun_out/r02c_topk_D.ncu-rep 2>&1 | tail -3
ls -la gpurun_out/r02c_topk_D.ncu-rep
