#!/bin/bash
cd "$(dirname "$0")/.."
for g in 8 16 32 64; do
  echo "EBV_GEMM_GROUP=$g"; EBV_GEMM_GROUP=$g timeout 300 python scripts/factor_time.py 32768 8192 --reps 3 2>&1 | grep '^{' | python3 -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print('   ', d['n'], '%.3f ms'%d['ms_median'])"
done
