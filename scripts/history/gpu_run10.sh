timeout -s KILL 300 python scripts/check_gemm.py 2>&1 | tail -6
timeout -s KILL 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest10.log 2>&1; tail -4 gpurun_out/pytest10.log
EBV_GEMM_TMA=0 timeout -s KILL 300 python scripts/gemm_bench.py > gpurun_out/gemm_bench_v10.log 2>&1; head -6 gpurun_out/gemm_bench_v10.log
timeout -s KILL 900 python bench.py --no-e2e > gpurun_out/bench10.log 2>&1; tail -c 1800 gpurun_out/bench10.log
