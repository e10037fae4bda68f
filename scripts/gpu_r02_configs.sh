#!/bin/bash
cd "$(dirname "$0")/.."
timeout 1200 python scripts/bench_configs.py > gpurun_out/r02_configs.jsonl 2> gpurun_out/r02_configs.err; echo "configs rc=$?"
timeout 900 python scripts/oracle_times.py > gpurun_out/r02_oracle_times.jsonl 2>&1; echo "oracle rc=$?"
cat gpurun_out/r02_oracle_times.jsonl
