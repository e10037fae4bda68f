timeout -s KILL 120 python scripts/debug_batched.py > gpurun_out/debug_batched.log 2>&1; cat gpurun_out/debug_batched.log | tail -20
timeout -s KILL 300 python scripts/gemm_bench.py > gpurun_out/gemm_bench.log 2>&1; cat gpurun_out/gemm_bench.log
timeout -s KILL 120 python scripts/prof_factor.py --n 4096 > gpurun_out/prof_plain.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv --log-file gpurun_out/launches_4096.csv python scripts/prof_factor.py --n 4096 --reps 1 > gpurun_out/ncu1.log 2>&1; tail -3 gpurun_out/ncu1.log; wc -l gpurun_out/launches_4096.csv
