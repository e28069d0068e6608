# prefill A/B, 10 steps (every chunk once), alternating
for V in 1 0 1 0 1 0; do
  if [ $V = 1 ]; then export RIKI_NO_PREFILL=1; else unset RIKI_NO_PREFILL; fi
  timeout 900 python bench.py --config 5 --steps 10 --warmup 3 --quick --no-cpu > gpurun_out/e13_np$V.log 2>&1
  echo "no_prefill=$V: $(tail -c 1500 gpurun_out/e13_np$V.log | grep -o '"value": [0-9.]*')"
done
