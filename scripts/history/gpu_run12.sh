timeout -s KILL 600 python -m pytest tests/test_gpu_dist.py -q --timeout 300 -p no:cacheprovider 2>&1 | tail -2
timeout -s KILL 900 python scripts/bench_configs.py > gpurun_out/configs12.jsonl 2>&1; cat gpurun_out/configs12.jsonl
