#!/bin/bash
export REGOT_B200_MAILBOX_TIMEOUT_S=30 REGOT_B200_PCG_BLOCKS_INFO=1
echo "== one cluster, 300x260"; timeout 60 python scripts/r2_blocks_dbg.py 300 260 2>&1 | tail -2
echo "== 14x9 clusters, 3000x2600"; REGOT_B200_PCG_BLOCKS_ONE_CLUSTER_ENTRIES=0 timeout 60 python scripts/r2_blocks_dbg.py 3000 2600 2>&1 | tail -2
echo "== 2x3 clusters, 300x260"; REGOT_B200_PCG_BLOCKS_GRID=2x3 timeout 60 python scripts/r2_blocks_dbg.py 300 260 2>&1 | tail -2
echo "== 1x2 cluster, 300x260"; REGOT_B200_PCG_BLOCKS_GRID=1x2 timeout 60 python scripts/r2_blocks_dbg.py 300 260 2>&1 | tail -2
echo "== L2 9x16, 300x260"; REGOT_B200_PCG_BLOCKS_CLUSTER=0 timeout 60 python scripts/r2_blocks_dbg.py 300 260 2>&1 | tail -2
