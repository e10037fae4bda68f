timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -k "not full_size and not c3 and not c4" > gpurun_out/pytest4.log 2>&1; tail -8 gpurun_out/pytest4.log
timeout -s KILL 120 python __graft_entry__.py > gpurun_out/smoke4.log 2>&1; tail -3 gpurun_out/smoke4.log
timeout -s KILL 300 python bench.py --n 8192 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench8192_4.log 2>&1; tail -c 1500 gpurun_out/bench8192_4.log
timeout -s KILL 600 python bench.py --steps 2 --warmup 3 > gpurun_out/bench32768_4.log 2>&1; tail -c 4000 gpurun_out/bench32768_4.log
timeout -s KILL 120 python scripts/prof_factor.py --n 4096 > gpurun_out/prof_plain4.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/launches_4096_v2.csv python scripts/prof_factor.py --n 4096 --reps 1 > gpurun_out/ncu4a.log 2>&1
timeout -s KILL 120 python scripts/prof_gemm.py --M 8192 --N 8192 --K 256 > gpurun_out/prof_gemm_plain.log 2>&1 && \
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:gemm_sub -s 1 -c 1 -o gpurun_out/gemm_8192_256 python scripts/prof_gemm.py --M 8192 --N 8192 --K 256 > gpurun_out/ncu4b.log 2>&1; tail -3 gpurun_out/ncu4b.log
