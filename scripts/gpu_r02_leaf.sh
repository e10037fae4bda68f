#!/bin/bash
cd "$(dirname "$0")/.."
for lf in 64 48 32; do for nb in 96 128 192; do
  r=$(( (nb + lf - 1) / lf * lf ))
  timeout 300 python scripts/factor_time.py 8192 --reps 4 --nb $r --leaf $lf 2>&1 | tail -1
done; done
for lf in 64 32; do timeout 300 python scripts/factor_time.py 4096 1024 --reps 4 --leaf $lf 2>&1 | tail -2; done
