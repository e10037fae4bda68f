#!/bin/bash
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for t in 0 4096 6144; do
    EBV_TAIL_ROWS=$t timeout 300 python scripts/factor_time.py 16384 32768 --reps 3 | cut -c1-60 | sed "s/^/tail=$t /"
  done
done
