#!/bin/bash
# the batched kernels' shuffle chunk (compile time): C5 timing per value
cd "$(dirname "$0")/.."
for ch in 8 4 6; do
  EBV_EXTRA_NVCC_FLAGS="-DEBV_BATCHED_CH=$ch" python -c "from paper_1907_05767_b200 import _build; _build.build(force=True)" > /dev/null 2>&1 || { echo "build $ch failed"; continue; }
  for i in 1 2; do
    timeout 300 python scripts/bench_batched.py --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('CH=$ch', d['ms'])"
  done
done
python -c "from paper_1907_05767_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
