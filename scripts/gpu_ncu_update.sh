# ncu --set full of the longest trailing-update launch of one n=32768 factorization
set -u
mkdir -p gpurun_out
timeout -s KILL 300 python scripts/prof_factor.py --n 32768 --reps 1 > gpurun_out/pf.log 2>&1 || exit 1
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_tma --csv \
  --log-file gpurun_out/gemm_launches.csv python scripts/prof_factor.py --n 32768 --reps 1 > /dev/null 2>&1
IDX=$(python - <<'PY'
import csv
rows=[r for r in csv.reader(l for l in open("gpurun_out/gemm_launches.csv") if l.startswith('"'))]
h=rows[0]; d=rows[1:]
iv=h.index("Metric Value")
vals=[float(r[iv].replace(",","")) for r in d]
print(max(range(len(vals)), key=lambda i: vals[i]))
PY
)
echo "longest gemm_tma launch index: $IDX"
timeout -s KILL 1200 ncu --set full --import-source on --clock-control none -k regex:gemm_tma -s $IDX -c 1 \
  -o gpurun_out/${REPORT:-r01_update_step0} -f python scripts/prof_factor.py --n 32768 --reps 1 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
