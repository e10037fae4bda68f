timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -k "not full_size and not c3 and not c4" > gpurun_out/pytest6.log 2>&1; tail -5 gpurun_out/pytest6.log
for v in 0 1 2; do echo "tma $v"; EBV_GEMM_TMA=$v timeout -s KILL 300 python scripts/gemm_bench.py > gpurun_out/gemm_bench_tma$v.log 2>&1; cat gpurun_out/gemm_bench_tma$v.log; done
timeout -s KILL 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench32768_6.log 2>&1; tail -c 2500 gpurun_out/bench32768_6.log
timeout -s KILL 120 python scripts/prof_gemm.py --M 16384 --N 16384 --K 256 > gpurun_out/prof_gemm_plain6.log 2>&1 && \
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tma -s 1 -c 1 -o gpurun_out/gemm_tma_16384_256 python scripts/prof_gemm.py --M 16384 --N 16384 --K 256 > gpurun_out/ncu6.log 2>&1; tail -2 gpurun_out/ncu6.log
