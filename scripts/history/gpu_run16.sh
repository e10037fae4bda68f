timeout -s KILL 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest16.log 2>&1; tail -3 gpurun_out/pytest16.log
timeout -s KILL 800 python scripts/sweep_nb.py 1024,8192,32768 2>&1 | tee gpurun_out/sweep16.jsonl
