# large-graph expansion occupancy: 6/5 blocks per SM (default) vs 5/5 (b5) vs 4/4 (b4)
for L in libriki.so libriki_b5.so libriki_b4.so libriki.so libriki_b5.so libriki_b4.so; do
  RIKI_LIB=$PWD/paper_2001_06770_b200/$L timeout 900 python bench.py --config 5 --steps 10 --warmup 3 --quick --no-cpu > gpurun_out/e22_c5_$L.log 2>&1
  echo "C5 $L: $(tail -c 1500 gpurun_out/e22_c5_$L.log | grep -o '"value": [0-9.]*')"
done
