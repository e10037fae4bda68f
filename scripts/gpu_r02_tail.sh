#!/bin/bash
# narrower (128-wide) panels once fewer than t rows remain (EBV_TAIL_ROWS)
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for t in 0 4096 8192 12288; do
    EBV_TAIL_ROWS=$t timeout 300 python scripts/factor_time.py 32768 --reps 3 | cut -c1-60 | sed "s/^/tail=$t /"
  done
done
