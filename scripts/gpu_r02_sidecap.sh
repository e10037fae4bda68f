#!/bin/bash
# side-stream GEMMs on at most g persistent CTAs (EBV_SIDE_GEMM_GRID)
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for g in 0 296 148 74; do
    EBV_SIDE_GEMM_GRID=$g timeout 300 python scripts/factor_time.py 8192 32768 --reps 3 | cut -c1-60 | sed "s/^/cap=$g /"
  done
done
