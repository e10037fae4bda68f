set -u
mkdir -p gpurun_out
timeout -s KILL 900 python bench.py > gpurun_out/bench22.log 2>&1; tail -1 gpurun_out/bench22.log | cut -c1-300
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench22_ref.log 2>&1; tail -1 gpurun_out/bench22_ref.log | cut -c1-300
timeout -s KILL 300 python __graft_entry__.py > gpurun_out/smoke22.log 2>&1; tail -2 gpurun_out/smoke22.log
timeout -s KILL 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches22.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu22.log 2>&1; wc -l gpurun_out/launches22.csv
