#!/bin/bash
cd "$(dirname "$0")/.."
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_variants.py -m gpu -x -q 2>&1 | tail -3
for rep in 1 2; do
  timeout 300 python scripts/factor_time.py 1024 8192 --reps 9 | cut -c1-60 | sed "s/^/blk /"
  EBV_PANEL_BLK=0 timeout 300 python scripts/factor_time.py 1024 8192 --reps 9 | cut -c1-60 | sed "s/^/old /"
done
