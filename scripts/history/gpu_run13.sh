timeout -s KILL 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest13.log 2>&1; tail -3 gpurun_out/pytest13.log
timeout -s KILL 900 python scripts/bench_configs.py > gpurun_out/configs13.jsonl 2>&1; cat gpurun_out/configs13.jsonl | cut -c1-220
timeout -s KILL 900 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench13.log 2>&1; tail -1 gpurun_out/bench13.log | cut -c1-700
timeout -s KILL 120 python scripts/prof_solve.py --n 8192 --nrhs 16 > /dev/null 2>&1 && timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:solve_kernel -s 2 -c 2 -o gpurun_out/solve16 python scripts/prof_solve.py --n 8192 --nrhs 16 > gpurun_out/ncu13a.log 2>&1; tail -1 gpurun_out/ncu13a.log
