# launch list of the bench command (shares of the step), then one full ncu capture of the dominant kernel
timeout -s KILL 600 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_for_ncu.log 2>&1 && \
timeout -s KILL 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_bench.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu9a.log 2>&1; tail -2 gpurun_out/ncu9a.log; wc -l gpurun_out/r01_launches_bench.csv
timeout -s KILL 120 python scripts/prof_factor.py --n 32768 --reps 1 > gpurun_out/prof_plain9.log 2>&1 && \
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:gemm_tma -s 16 -c 1 -o gpurun_out/r01_gemm_tma_in_factor python scripts/prof_factor.py --n 32768 --reps 1 > gpurun_out/ncu9b.log 2>&1; tail -2 gpurun_out/ncu9b.log
