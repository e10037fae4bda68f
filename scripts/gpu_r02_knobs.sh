#!/bin/bash
cd "$(dirname "$0")/.."
run() { echo "$1"; env $1 timeout 300 python scripts/factor_time.py 8192 1024 --reps 4 2>&1 | grep '^{' | python3 -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print('   ', d['n'], '%.3f ms'%d['ms_median'])"; }
run "X=0"
run "EBV_TAIL_ROWS=2048"
run "EBV_TAIL_ROWS=4096"
run "EBV_PANEL_FUSED_ROWS=2048"
run "EBV_PANEL_FUSED_ROWS=100000"
run "EBV_TRSM_LLU_CC=1"
run "EBV_TRSM_LLU_CC=4"
run "EBV_U12_SPLIT_ROWS=100000"
run "EBV_GEMM_TMA=5"
run "EBV_GEMM_TMA=3"
