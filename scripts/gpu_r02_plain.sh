#!/bin/bash
# the lane-level EbV pairing (two systems per warp, rows t and 31-t) against
# one system per warp (lane = row), same scheme otherwise: parity, then C5
cd "$(dirname "$0")/.."
EBV_BATCHED_PLAIN=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -m gpu -x -q -k "batched" 2>&1 | tail -1
for i in 1 2; do
  for v in 0 1; do
    EBV_BATCHED_PLAIN=$v timeout 300 python scripts/bench_batched.py --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('plain=$v', d['ms'], d['gbs_aggregate'])"
  done
done
