#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_solve_chain.py -q -x -p no:cacheprovider > gpurun_out/solve_chain_tests.log 2>&1
echo "chain tests rc=$?"; tail -3 gpurun_out/solve_chain_tests.log
timeout 300 python scripts/bench_solve.py 1024x1 8192x1 8192x16 32768x1 > gpurun_out/bench_solve_chain.jsonl 2>&1; echo "bench chain rc=$?"
cat gpurun_out/bench_solve_chain.jsonl
timeout 300 python scripts/bench_solve.py 8192x1 > /dev/null 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:solve_chain --csv python scripts/bench_solve.py 8192x1 > gpurun_out/ncu_solve_chain_8192.csv 2>&1
echo "ncu rc=$?"; grep solve_chain gpurun_out/ncu_solve_chain_8192.csv | awk -F'","' '{print $5, $NF}' | head -6
