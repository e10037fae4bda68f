#!/bin/bash
cd "$(dirname "$0")/.."
timeout 300 python scripts/bench_solve.py 8192x1 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:solve_chain_kernel -s 2 -c 2 -o gpurun_out/solve_chain_8192 python scripts/bench_solve.py 8192x1 > gpurun_out/ncu_chain.log 2>&1
echo "ncu rc=$?"; tail -5 gpurun_out/ncu_chain.log
