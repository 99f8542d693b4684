#!/bin/bash
# first solve of a fresh context at config D (buffers grow from refresh to refresh) against the second one
REPS=1 timeout 600 python scripts/solve_cloud.py D 0 2>&1 | grep -E "wall_s" | cut -c1-120
REPS=2 timeout 600 python scripts/solve_cloud.py D 0 2>&1 | grep -E "wall_s" | cut -c1-120
