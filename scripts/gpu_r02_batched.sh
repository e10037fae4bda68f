#!/bin/bash
# batched n = 32 kernel: parity tests, then C5 timing of the round-1 kernel
# (EBV_BATCHED_V1=0) against the current default, alternating
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -m gpu -x -q -k "batched or forced" 2>&1 | tail -5
for i in 1 2; do
  for v in 0 1; do
    EBV_BATCHED_V1=$v timeout 300 python scripts/bench_batched.py --steps 20 | sed "s/^/v1=$v /"
  done
done
