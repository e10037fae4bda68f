timeout -s KILL 120 python scripts/prof_factor.py --n 32768 --reps 1 > gpurun_out/prof_plain17.log 2>&1 && \
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:gemm_tma -s 32 -c 1 -o gpurun_out/r01_gemm_tma_trailing_big python scripts/prof_factor.py --n 32768 --reps 1 > gpurun_out/ncu17.log 2>&1; tail -2 gpurun_out/ncu17.log
