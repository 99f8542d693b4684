#!/bin/bash
# ELL stream of the panel mat-vec: tests, then config D with the stream on / off
timeout 600 python -m pytest tests/test_sparse_gpu.py -x -q -m gpu 2>&1 | tail -5
REPS=2 timeout 600 python scripts/solve_cloud.py D 0 2>&1 | tail -9
REGOT_B200_PANEL_ELL=0 REPS=2 timeout 600 python scripts/solve_cloud.py D 0 2>&1 | tail -9
