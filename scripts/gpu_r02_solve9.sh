#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_solve_chain.py tests/test_gpu_edge.py -m gpu -x -q -k "chain or trsm or blocked" 2>&1 | tail -2
timeout 600 python scripts/bench_solve.py 32768x1 32768x1 8192x16 8192x1 1024x1 2>&1 | grep "^{" | cut -c1-200
./probes/chain_trace 32768 > gpurun_out/ct32768b.txt 2>&1; sed -n 3p gpurun_out/ct32768b.txt; sed -n 40,44p gpurun_out/ct32768b.txt
