# exact arena allocation of the memoised predecessor lists: parity, config-3 chunking, A/B at configs 2 and 5
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_chunking.py tests/test_gpu_tie_break.py tests/test_gpu_boundary.py -q -x -p no:cacheprovider > gpurun_out/e15_tests.log 2>&1; tail -2 gpurun_out/e15_tests.log
timeout 900 python bench.py --config 3 --steps 3 --warmup 2 --quick --no-cpu > gpurun_out/e15_c3.log 2>&1
echo "C3: $(tail -c 1500 gpurun_out/e15_c3.log | grep -o '"value": [0-9.]*\|"retries": [0-9]*\|"reallocs": [0-9]*' | tr '\n' ' ')"
RIKI_LIB=$PWD/paper_2001_06770_b200/libriki_base.so timeout 900 python bench.py --config 3 --steps 3 --warmup 2 --quick --no-cpu > gpurun_out/e15_c3_base.log 2>&1
echo "C3 base: $(tail -c 1500 gpurun_out/e15_c3_base.log | grep -o '"value": [0-9.]*\|"retries": [0-9]*\|"reallocs": [0-9]*' | tr '\n' ' ')"
for L in libriki_base.so libriki.so libriki_base.so libriki.so; do
  RIKI_LIB=$PWD/paper_2001_06770_b200/$L timeout 600 python bench.py --config 2 --steps 20 --warmup 3 --quick --no-cpu > gpurun_out/e15_c2_$L.log 2>&1
  echo "C2 $L: $(tail -c 1500 gpurun_out/e15_c2_$L.log | grep -o '"value": [0-9.]*')"
done
