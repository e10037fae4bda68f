#!/bin/bash
cd "$(dirname "$0")/.."
for v in 8192 4096 2048 1024 512; do
  echo "EBV_PANEL_FUSED_ROWS=$v"; EBV_PANEL_FUSED_ROWS=$v timeout 300 python scripts/factor_time.py 32768 16384 8192 4096 --reps 3 2>&1 | grep '^{' | python3 -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print('   ', d['n'], '%.3f ms'%d['ms_median'])"
done
