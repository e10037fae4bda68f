#!/bin/bash
cd "$(dirname "$0")/.."
EBV_SOLVE_CHAIN=2 timeout 600 python -m pytest tests/test_gpu_solve_chain.py tests/test_gpu_parity.py -k "solve" -q -x -p no:cacheprovider > gpurun_out/solve_chain_tests.log 2>&1
echo "chain tests rc=$?"; tail -2 gpurun_out/solve_chain_tests.log
C="8192x1 8192x4 8192x8 8192x16 32768x1 32768x4 32768x16 4096x16 2048x16"
EBV_SOLVE_CHAIN=2 timeout 600 python scripts/bench_solve.py $C > gpurun_out/r02_solve_chain_groups.jsonl 2>&1; echo "chain rc=$?"
python - <<'PY'
import json
for l in open('gpurun_out/r02_solve_chain_groups.jsonl'):
    if l.startswith('{'):
        x=json.loads(l); print(x['n'],x['nrhs'],'chain %.3f'%x['ms'])
PY
