# cost of the device atomics counter (libriki.so) vs the build before it (libriki_base.so)
for L in libriki_base.so libriki.so libriki_base.so libriki.so libriki_base.so libriki.so; do
  RIKI_LIB=$PWD/paper_2001_06770_b200/$L timeout 600 python bench.py --config 2 --steps 20 --warmup 3 --quick --no-cpu > gpurun_out/e16_c2_$L.log 2>&1
  echo "C2 $L: $(tail -c 1500 gpurun_out/e16_c2_$L.log | grep -o '"value": [0-9.]*')"
done
for L in libriki_base.so libriki.so libriki_base.so libriki.so; do
  RIKI_LIB=$PWD/paper_2001_06770_b200/$L timeout 900 python bench.py --config 3 --steps 3 --warmup 2 --quick --no-cpu > gpurun_out/e16_c3_$L.log 2>&1
  echo "C3 $L: $(tail -c 1500 gpurun_out/e16_c3_$L.log | grep -o '"value": [0-9.]*')"
done
