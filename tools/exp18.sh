# push fast path (uniform slot, skip empty unrolled pushes) + cheaper identification test: parity, A/B vs the previous build
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wikidata_scale.py tests/test_vertex_partitioned.py tests/test_gpu_tie_break.py -q -x -p no:cacheprovider > gpurun_out/e18_tests.log 2>&1; tail -2 gpurun_out/e18_tests.log
for L in libriki_prev.so libriki.so libriki_prev.so libriki.so libriki_prev.so libriki.so; do
  RIKI_LIB=$PWD/paper_2001_06770_b200/$L timeout 600 python bench.py --config 2 --steps 20 --warmup 3 --quick --no-cpu > gpurun_out/e18_c2_$L.log 2>&1
  echo "C2 $L: $(tail -c 1500 gpurun_out/e18_c2_$L.log | grep -o '"value": [0-9.]*')"
done
for L in libriki_prev.so libriki.so libriki_prev.so libriki.so; do
  RIKI_LIB=$PWD/paper_2001_06770_b200/$L timeout 900 python bench.py --config 5 --steps 10 --warmup 3 --quick --no-cpu > gpurun_out/e18_c5_$L.log 2>&1
  echo "C5 $L: $(tail -c 1500 gpurun_out/e18_c5_$L.log | grep -o '"value": [0-9.]*')"
done
