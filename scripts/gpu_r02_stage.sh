#!/bin/bash
cd "$(dirname "$0")/.."
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_variants.py tests/test_gpu_band.py -m gpu -x -q 2>&1 | tail -1
for rep in 1 2; do timeout 300 python scripts/factor_time.py 1024 8192 --reps 9 | cut -c1-60; done
timeout 300 python scripts/factor_time.py 32768 --reps 3 | cut -c1-60
timeout 300 python scripts/update_insitu.py --n 32768 | cut -c1-400
