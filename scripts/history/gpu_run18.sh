set -u
mkdir -p gpurun_out
timeout -s KILL 900 python bench.py > gpurun_out/bench18.log 2>&1; tail -1 gpurun_out/bench18.log | cut -c1-400
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches18.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu18a.log 2>&1; tail -2 gpurun_out/ncu18a.log | cut -c1-300; wc -l gpurun_out/launches18.csv
timeout -s KILL 120 python scripts/prof_factor.py --n 32768 --reps 1 > gpurun_out/prof_plain18.log 2>&1 && \
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:gemm_tma -s 0 -c 1 -o gpurun_out/r01_gemm_tma_nb512_step0 python scripts/prof_factor.py --n 32768 --reps 1 > gpurun_out/ncu18b.log 2>&1; tail -2 gpurun_out/ncu18b.log
