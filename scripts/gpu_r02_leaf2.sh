#!/bin/bash
# diagonal-block leaf with published reciprocals + Markstein quotients:
# parity, then factor times at GD = 4 (built) and GD = 8 (rebuilt here)
cd "$(dirname "$0")/.."
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_variants.py -m gpu -x -q 2>&1 | tail -2
for rep in 1 2; do timeout 300 python scripts/factor_time.py 1024 8192 --reps 9 | sed "s/^/G4 /" | cut -c1-80; done
timeout 300 python scripts/factor_time.py 32768 --reps 3 | sed "s/^/G4 /" | cut -c1-80
EBV_EXTRA_NVCC_FLAGS=-DEBV_LEAF_G=8 python -c "from paper_1907_05767_b200 import _build; _build.build(force=True)" && echo rebuilt-G8
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -m gpu -x -q 2>&1 | tail -2
for rep in 1 2; do timeout 300 python scripts/factor_time.py 1024 8192 --reps 9 | sed "s/^/G8 /" | cut -c1-80; done
timeout 300 python scripts/factor_time.py 32768 --reps 3 | sed "s/^/G8 /" | cut -c1-80
