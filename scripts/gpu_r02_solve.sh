#!/bin/bash
# chain solve: parity first (short timeouts), then timings chain vs wavefront
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_solve_chain.py -q -x -p no:cacheprovider > gpurun_out/solve_chain_tests.log 2>&1
echo "chain tests rc=$?"; tail -15 gpurun_out/solve_chain_tests.log
timeout 300 python scripts/bench_solve.py > gpurun_out/bench_solve_chain.jsonl 2>&1; echo "bench chain rc=$?"
EBV_SOLVE_CHAIN=0 timeout 300 python scripts/bench_solve.py > gpurun_out/bench_solve_wave.jsonl 2>&1; echo "bench wave rc=$?"
cat gpurun_out/bench_solve_chain.jsonl gpurun_out/bench_solve_wave.jsonl
