#!/bin/bash
cd "$(dirname "$0")/.."
for v in base fwd; do echo "== $v"; timeout 60 ./probes/chain_trace_$v 8192 > gpurun_out/ct_$v.txt 2>&1; sed -n "2,3p;28,32p" gpurun_out/ct_$v.txt; done
timeout 600 python -m pytest tests/test_gpu_solve_chain.py -q -x -p no:cacheprovider > gpurun_out/solve_chain_tests.log 2>&1
echo "chain tests rc=$?"; tail -2 gpurun_out/solve_chain_tests.log
timeout 300 python scripts/bench_solve.py 1024x1 8192x1 8192x4 32768x1 32768x4 32768x16 > gpurun_out/bench_solve_chain.jsonl 2>&1; echo "bench chain rc=$?"
cat gpurun_out/bench_solve_chain.jsonl | cut -c1-80
