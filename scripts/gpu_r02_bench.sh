#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-dist-n1 > gpurun_out/bench_short.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-dist-n1 > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?"
