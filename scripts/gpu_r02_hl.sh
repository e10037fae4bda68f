#!/bin/bash
# the chain solve's helper lag HL (compile time) re-swept with the final code
cd "$(dirname "$0")/.."
for hl in 5 4 6; do
  EBV_EXTRA_NVCC_FLAGS="-DEBV_CHAIN_HL=$hl" python -c "from paper_1907_05767_b200 import _build; _build.build(force=True)" > /dev/null 2>&1 || { echo "build $hl failed"; continue; }
  timeout 300 python scripts/bench_solve.py 32768x1 32768x1 8192x16 8192x1 2>&1 | grep "^{" | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l); print('HL=$hl', d['n'], d['nrhs'], round(d['ms'],3))"
done
python -c "from paper_1907_05767_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
