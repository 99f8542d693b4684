#!/bin/bash
# kernel-by-kernel PCG after a change: the tests that drive it (one GPU and loopback-sharded), then config D
mkdir -p gpurun_out
export REGOT_B200_MAILBOX_TIMEOUT_S=120
timeout 900 python -m pytest tests/test_sparse_gpu.py tests/test_pcg_blocks_gpu.py tests/test_sharded_loopback_gpu.py tests/test_pointcloud_gpu.py -q -x 2>&1 | tail -8 | tee gpurun_out/mk_pytest.txt
REPS=2 timeout 600 python scripts/solve_cloud.py D 0 2>&1 | tail -12 | tee gpurun_out/mk_D.txt
