# large-graph expansion occupancy: 4 (b4) vs 3 (b3) vs 2 (b2) blocks per SM
for L in libriki_b4.so libriki_b3.so libriki_b2.so libriki_b4.so libriki_b3.so libriki_b2.so; do
  RIKI_LIB=$PWD/paper_2001_06770_b200/$L timeout 900 python bench.py --config 5 --steps 10 --warmup 3 --quick --no-cpu > gpurun_out/e23_c5_$L.log 2>&1
  echo "C5 $L: $(tail -c 1500 gpurun_out/e23_c5_$L.log | grep -o '"value": [0-9.]*')"
done
for L in libriki_b4.so libriki_b3.so; do
  RIKI_LIB=$PWD/paper_2001_06770_b200/$L timeout 900 python bench.py --config 3 --steps 3 --warmup 2 --quick --no-cpu > gpurun_out/e23_c3_$L.log 2>&1
  echo "C3 $L: $(tail -c 1500 gpurun_out/e23_c3_$L.log | grep -o '"value": [0-9.]*')"
done
