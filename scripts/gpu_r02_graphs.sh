#!/bin/bash
cd "$(dirname "$0")/.."
for args in "--graphs 1" "--graphs 0"; do
  timeout 300 python scripts/factor_time.py 32768 16384 8192 4096 --reps 4 $args 2>&1 | tail -4
done
EBV_GRAPH_PRIO=0 timeout 300 python scripts/factor_time.py 16384 4096 --reps 4 2>&1 | tail -2
