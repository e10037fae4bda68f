timeout -s KILL 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest15.log 2>&1; tail -3 gpurun_out/pytest15.log
timeout -s KILL 900 python scripts/bench_configs.py > gpurun_out/configs15.jsonl 2>&1; cat gpurun_out/configs15.jsonl | cut -c1-200
timeout -s KILL 900 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench15.log 2>&1; tail -1 gpurun_out/bench15.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ['value','factor_ms','solve_ms','correct']})"
