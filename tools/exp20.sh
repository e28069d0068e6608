# BIG-graph expansion occupancy (6 blocks/SM for 16/32-bit rows, 5 for 64-bit, grids of one wave) vs RIKI_NO_BIGOCC=1
timeout 1500 python -m pytest tests/test_gpu_wikidata_scale.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/e20_tests.log 2>&1; tail -1 gpurun_out/e20_tests.log
for V in 1 0 1 0 1 0; do
  if [ $V = 1 ]; then export RIKI_NO_BIGOCC=1; else unset RIKI_NO_BIGOCC; fi
  timeout 900 python bench.py --config 5 --steps 10 --warmup 3 --quick --no-cpu > gpurun_out/e20_c5_nb$V.log 2>&1
  echo "C5 no_bigocc=$V: $(tail -c 1500 gpurun_out/e20_c5_nb$V.log | grep -o '"value": [0-9.]*')"
done
unset RIKI_NO_BIGOCC
for i in 1 2; do
  timeout 600 python bench.py --config 2 --steps 20 --warmup 3 --quick --no-cpu > gpurun_out/e20_c2_$i.log 2>&1
  echo "C2: $(tail -c 1500 gpurun_out/e20_c2_$i.log | grep -o '"value": [0-9.]*')"
done
