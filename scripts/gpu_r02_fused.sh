#!/bin/bash
# panel rows up to which the fused (blocked) panel-leaf kernel runs
cd "$(dirname "$0")/.."
for rows in 2048 4096 8192 16384; do
  EBV_PANEL_FUSED_ROWS=$rows timeout 300 python scripts/factor_time.py 8192 --reps 9 | cut -c1-60 | sed "s/^/rows=$rows /"
done
for rows in 4096 8192 32768; do
  EBV_PANEL_FUSED_ROWS=$rows timeout 300 python scripts/factor_time.py 32768 --reps 3 | cut -c1-60 | sed "s/^/rows=$rows /"
done
