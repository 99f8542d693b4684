#!/bin/bash
# whole GPU suite (hang-proof: the host mailbox gives up after 60 s), then per-iteration times of the direction solve
mkdir -p gpurun_out
export REGOT_B200_MAILBOX_TIMEOUT_S=60
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 | tee gpurun_out/pytest_gpu.txt
bash scripts/r2_blocks_iter.sh > /dev/null 2>&1; cat gpurun_out/blocks_iter.txt
