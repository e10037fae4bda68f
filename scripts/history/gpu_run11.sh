timeout -s KILL 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest11.log 2>&1; tail -15 gpurun_out/pytest11.log
timeout -s KILL 900 python bench.py > gpurun_out/bench11.log 2>&1; tail -c 600 gpurun_out/bench11.log
timeout -s KILL 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench11_ref.log 2>&1; tail -c 800 gpurun_out/bench11_ref.log
