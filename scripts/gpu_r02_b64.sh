#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -m gpu -x -q -k "batched or forced" 2>&1 | tail -1
for i in 1 2; do
  timeout 300 python scripts/bench_batched.py --n 64 --steps 10 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('n64', d['ms'], d['gbs_aggregate'])"
  timeout 300 python scripts/bench_batched.py --n 48 --steps 10 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('n48', d['ms'], d['gbs_aggregate'])"
done
