# C5: global-scratch recovery CTAs (RIKI_BIG_CTAS) A/B, quick bench
for B in 2 8 16 2 8; do
  RIKI_BIG_CTAS=$B timeout 900 python bench.py --config 5 --steps 4 --warmup 2 --quick --no-cpu > gpurun_out/e5_big$B.log 2>&1
  echo "big $B: $(tail -c 900 gpurun_out/e5_big$B.log | grep -o '"value": [0-9.]*')"
done
