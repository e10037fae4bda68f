set -u
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -k "block_width" 2>&1 | tail -1
timeout -s KILL 600 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench19_plain.log 2>&1; tail -1 gpurun_out/bench19_plain.log | cut -c1-200
timeout -s KILL 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches19.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu19.log 2>&1; tail -1 gpurun_out/ncu19.log | cut -c1-300; wc -l gpurun_out/launches19.csv
