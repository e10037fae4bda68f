#!/bin/bash
# round-2 closing run: smoke, the whole GPU suite, the bench line (both
# arms), the config table, the batched kernel's ncu capture and the bench's
# launch list
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --maxfail=40 -rf > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"
timeout 1200 python scripts/bench_configs.py > gpurun_out/r02_configs.jsonl 2> gpurun_out/r02_configs.err; echo "configs rc=$?"
timeout 300 python scripts/ncu_target.py batched > gpurun_out/plain_batched.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:batched1_kernel -s 1 -c 1 -o gpurun_out/r02_ncu_batched1 python scripts/ncu_target.py batched > gpurun_out/ncu_batched.log 2>&1; echo "ncu batched rc=$?"
timeout 600 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-dist-n1 > gpurun_out/bench_short.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-dist-n1 > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?"
