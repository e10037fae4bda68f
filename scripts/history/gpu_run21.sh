set -u
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py -q -x -k "dist or solve" 2>&1 | tail -3
timeout -s KILL 600 python bench.py --force-dist --nb 256 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench21_dist.log 2>&1; tail -1 gpurun_out/bench21_dist.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d.get(k) for k in ['value','factor_ms','solve_ms','correct','gpu_launches']}, d['config']['path'])" || tail -5 gpurun_out/bench21_dist.log
timeout -s KILL 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench21.log 2>&1; tail -1 gpurun_out/bench21.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d.get(k) for k in ['value','factor_ms','solve_ms','correct','gpu_launches']}, d['config']['path'])" || tail -5 gpurun_out/bench21.log
