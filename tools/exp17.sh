# atomics counted only in profiling mode: production A/B at config 2 vs the pre-counter build; counter test; C5 profiling pass
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "counters or hitting_levels_random or search_random_small" -p no:cacheprovider > gpurun_out/e17_tests.log 2>&1; tail -2 gpurun_out/e17_tests.log
for L in libriki_base.so libriki.so libriki_base.so libriki.so; do
  RIKI_LIB=$PWD/paper_2001_06770_b200/$L timeout 600 python bench.py --config 2 --steps 20 --warmup 3 --quick --no-cpu > gpurun_out/e17_c2_$L.log 2>&1
  echo "C2 $L: $(tail -c 1500 gpurun_out/e17_c2_$L.log | grep -o '"value": [0-9.]*')"
done
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu > gpurun_out/e17_c5.log 2>&1
tail -c 3000 gpurun_out/e17_c5.log | grep -o '"value": [0-9.]*\|"random_access_roofline": {[^}]*}'
