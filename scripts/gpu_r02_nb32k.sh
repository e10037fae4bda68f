#!/bin/bash
# block width at n = 32768 with the round-2 kernels (tail narrowing on)
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for nb in 512 384 448 640; do
    timeout 300 python scripts/factor_time.py 32768 --reps 3 --nb $nb | cut -c1-60 | sed "s/^/nb=$nb /"
  done
done
