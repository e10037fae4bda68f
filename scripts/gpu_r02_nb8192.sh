#!/bin/bash
# block width at n = 8192 (graph replay): 128 (default) vs 192 / 256 / 64
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for nb in 128 192 256 64; do
    timeout 300 python scripts/factor_time.py 8192 --reps 9 --nb $nb | sed "s/^/nb=$nb /"
  done
done
