#!/bin/bash
cd "$(dirname "$0")/.."
run() { echo "$1 $2"; env $1 timeout 300 python scripts/factor_time.py 8192 16384 --reps 4 $2 2>&1 | grep '^{' | python3 -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print('   ', d['n'], '%.3f ms'%d['ms_median'])"; }
run "X=0" ""
run "EBV_TRSM_LLU_GRID=296" ""
run "EBV_TRSM_LLU_GRID=148" ""
run "EBV_U12_LA=0" ""
run "X=0" "--nb 192"
run "EBV_PANEL_FUSED_ROWS=3072" ""
run "EBV_PANEL_FUSED_ROWS=6144" ""
