#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_solve_chain.py -q -x -p no:cacheprovider > gpurun_out/solve_chain_tests.log 2>&1
echo "chain tests rc=$?"; tail -2 gpurun_out/solve_chain_tests.log
C="1024x1 4096x1 8192x1 8192x2 8192x4 8192x8 8192x16 32768x1 32768x2 32768x4 32768x8 32768x16"
timeout 600 python scripts/bench_solve.py $C > gpurun_out/r02_solve_chain.jsonl 2>&1; echo "chain rc=$?"
EBV_SOLVE_CHAIN=0 timeout 600 python scripts/bench_solve.py $C > gpurun_out/r02_solve_wave.jsonl 2>&1; echo "wave rc=$?"
python - <<'PY'
import json
a=[json.loads(l) for l in open('gpurun_out/r02_solve_chain.jsonl') if l.startswith('{')]
b=[json.loads(l) for l in open('gpurun_out/r02_solve_wave.jsonl') if l.startswith('{')]
for x,y in zip(a,b): print(x['n'],x['nrhs'],'chain %.3f'%x['ms'],'wave %.3f'%y['ms'])
PY
