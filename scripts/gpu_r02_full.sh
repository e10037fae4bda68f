#!/bin/bash
# round 2: full GPU test suite, bench line, ncu evidence for the solve /
# batched / vector kernels (row d' of the verdict), launch list of the bench
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --maxfail=40 -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
for c in solve32768 solve8192x16 batched vector; do
  timeout 300 python scripts/ncu_target.py $c > gpurun_out/plain_$c.log 2>&1 || { echo "plain $c failed"; continue; }
done
K_solve32768="regex:solve_chain_kernel"; K_solve8192x16="regex:solve_chain_kernel"; K_batched="regex:batched_kernel"; K_vector="regex:vector_lu_kernel"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:solve_chain_kernel -s 2 -c 2 -o gpurun_out/r02_ncu_solve32768 python scripts/ncu_target.py solve32768 > gpurun_out/ncu_solve32768.log 2>&1; echo "ncu solve rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:solve_chain_kernel -s 2 -c 2 -o gpurun_out/r02_ncu_solve8192x16 python scripts/ncu_target.py solve8192x16 > gpurun_out/ncu_solve8192x16.log 2>&1; echo "ncu solve16 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:batched_kernel -s 1 -c 1 -o gpurun_out/r02_ncu_batched python scripts/ncu_target.py batched > gpurun_out/ncu_batched.log 2>&1; echo "ncu batched rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:vector_lu_kernel -s 1 -c 1 -o gpurun_out/r02_ncu_vector python scripts/ncu_target.py vector > gpurun_out/ncu_vector.log 2>&1; echo "ncu vector rc=$?"
