#!/bin/bash
cd "$(dirname "$0")/.."
C="32768x1 32768x1 8192x32 8192x64 8192x128 8192x256 32768x32 32768x64"
EBV_SOLVE_CHAIN=2 EBV_SOLVE_TRSM_RHS=100000 timeout 900 python scripts/bench_solve.py $C > gpurun_out/r02_solve_chain_many.jsonl 2>&1; echo "chain rc=$?"
EBV_SOLVE_TRSM_RHS=1 timeout 900 python scripts/bench_solve.py 8192x32 8192x64 8192x128 8192x256 32768x32 32768x64 > gpurun_out/r02_solve_trsm_many.jsonl 2>&1; echo "trsm rc=$?"
python - <<'PY'
import json
for f in ('gpurun_out/r02_solve_chain_many.jsonl','gpurun_out/r02_solve_trsm_many.jsonl'):
  for l in open(f):
    if l.startswith('{'):
        x=json.loads(l); print(f.split('_')[-2], x['n'],x['nrhs'],'%.3f'%x['ms'])
PY
