timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -k "not full_size and not c3 and not c4" > gpurun_out/pytest5.log 2>&1; tail -5 gpurun_out/pytest5.log
for c in 0 1 2 3; do echo "cfg $c"; EBV_GEMM_CFG=$c timeout -s KILL 300 python scripts/gemm_bench.py > gpurun_out/gemm_bench_cfg$c.log 2>&1; cat gpurun_out/gemm_bench_cfg$c.log; done
timeout -s KILL 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench32768_5.log 2>&1; tail -c 2500 gpurun_out/bench32768_5.log
timeout -s KILL 120 python scripts/prof_factor.py --n 1024 > gpurun_out/prof_plain5.log 2>&1 && \
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:"trsm|leaf" -s 3 -c 3 -o gpurun_out/leaf_1024 python scripts/prof_factor.py --n 1024 --reps 1 > gpurun_out/ncu5.log 2>&1; tail -3 gpurun_out/ncu5.log
