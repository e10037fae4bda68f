cd /root/repo
for rep in 1 2; do
  timeout 300 python scripts/factor_time.py 1024 8192 --reps 9 | cut -c1-60 | sed "s/^/blk /"
done
