timeout -s KILL 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest8.log 2>&1; tail -8 gpurun_out/pytest8.log
timeout -s KILL 120 python __graft_entry__.py > gpurun_out/smoke8.log 2>&1; tail -2 gpurun_out/smoke8.log
timeout -s KILL 900 python bench.py > gpurun_out/bench8.log 2>&1; tail -c 5000 gpurun_out/bench8.log
