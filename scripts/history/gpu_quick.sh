set -x
nvidia-smi -L
timeout -s KILL 600 python -m pytest tests -m gpu -x -q --timeout 240 -p no:cacheprovider -k "not full_size and not c3 and not c4" 2>&1 | tail -30 > gpurun_out/pytest_quick.log
tail -30 gpurun_out/pytest_quick.log
timeout -s KILL 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; tail -5 gpurun_out/smoke.log
timeout -s KILL 300 python bench.py --n 8192 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench8192.log 2>&1; tail -c 3000 gpurun_out/bench8192.log
