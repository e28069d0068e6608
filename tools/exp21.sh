# BIG-graph expansion: unroll 4 (heavy 3) at 6/5 blocks (u4) and at 5/4 blocks (u4m5) vs the default (unroll 3 / heavy 2)
for L in libriki.so libriki_u4.so libriki_u4m5.so libriki.so libriki_u4.so libriki_u4m5.so; do
  RIKI_LIB=$PWD/paper_2001_06770_b200/$L timeout 900 python bench.py --config 5 --steps 10 --warmup 3 --quick --no-cpu > gpurun_out/e21_c5_$L.log 2>&1
  echo "C5 $L: $(tail -c 1500 gpurun_out/e21_c5_$L.log | grep -o '"value": [0-9.]*')"
done
