# run 2's H fill overlapped with run 1 on a side stream: A/B (RIKI_NO_PREFILL=1 = fill in line) + parity
for V in 1 0 1 0; do
  if [ $V = 1 ]; then export RIKI_NO_PREFILL=1; else unset RIKI_NO_PREFILL; fi
  timeout 900 python bench.py --config 5 --steps 4 --warmup 2 --quick --no-cpu > gpurun_out/e12_np$V.log 2>&1
  echo "no_prefill=$V: $(tail -c 900 gpurun_out/e12_np$V.log | grep -o '"value": [0-9.]*')"
done
unset RIKI_NO_PREFILL
for V in 1 0; do
  if [ $V = 1 ]; then export RIKI_NO_PREFILL=1; else unset RIKI_NO_PREFILL; fi
  timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --quick --no-cpu > gpurun_out/e12_c2_np$V.log 2>&1
  echo "C2 no_prefill=$V: $(tail -c 900 gpurun_out/e12_c2_np$V.log | grep -o '"value": [0-9.]*')"
done
unset RIKI_NO_PREFILL
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wikidata_scale.py tests/test_gpu_chunking.py tests/test_gpu_boundary.py -q -x -p no:cacheprovider > gpurun_out/e12_tests.log 2>&1; tail -3 gpurun_out/e12_tests.log
