#!/bin/bash
cd "$(dirname "$0")/.."
for la in 0 1; do for nb in 64 128 192 256; do
  EBV_U12_LA=$la timeout 300 python scripts/factor_time.py 8192 --reps 4 --nb $nb 2>&1 | tail -1
done; done
for la in 0 1; do for nb in 256 384 512; do
  EBV_U12_LA=$la timeout 300 python scripts/factor_time.py 16384 --reps 3 --nb $nb 2>&1 | tail -1
done; done
for nb in 384 512 640 768; do
  timeout 300 python scripts/factor_time.py 32768 --reps 3 --nb $nb 2>&1 | tail -1
done
