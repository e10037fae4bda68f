#!/bin/bash
# round 2: full GPU test suite, then the default bench line
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --maxfail=40 -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
tail -40 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"
tail -5 gpurun_out/bench.err
