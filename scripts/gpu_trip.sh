#!/bin/bash
for dbg in 6 7; do
  echo "=== PCG_DBG=$dbg"; REGOT_B200_PCG_DBG=$dbg MAXIT=3 timeout 300 python scripts/solve_config.py B 2>&1 | grep -E "pcg " | tail -1
done
timeout 600 python scripts/solve_config.py B 0 1e-6 2>&1 | grep -E "rep|pcg" 
timeout 600 python scripts/solve_config.py B 0 1e-6 2>&1 | grep -E "rep|pcg" 
