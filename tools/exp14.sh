# new counter test; u64 expansion occupancy A/B (EXP_MINB64 6 = default, 5, 4)
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "counters" -p no:cacheprovider > gpurun_out/e14_tests.log 2>&1; tail -2 gpurun_out/e14_tests.log
for L in libriki.so libriki_m5.so libriki_m4.so libriki.so libriki_m5.so libriki_m4.so; do
  RIKI_LIB=$PWD/paper_2001_06770_b200/$L timeout 900 python bench.py --config 5 --steps 10 --warmup 3 --quick --no-cpu > gpurun_out/e14_$L.log 2>&1
  echo "$L: $(tail -c 1500 gpurun_out/e14_$L.log | grep -o '"value": [0-9.]*')"
done
