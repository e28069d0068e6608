# expansion occupancy: EXP_MINB 8 (32 regs, default) vs 6 (40 regs, u16/u32 rows); EXP_MINB64 6 (default) vs 5 (u64 rows)
for L in libriki.so libriki_b6.so libriki_m5.so libriki.so libriki_b6.so libriki_m5.so; do
  RIKI_LIB=$PWD/paper_2001_06770_b200/$L timeout 600 python bench.py --config 2 --steps 20 --warmup 3 --quick --no-cpu > gpurun_out/e19_c2_$L.log 2>&1
  echo "C2 $L: $(tail -c 1500 gpurun_out/e19_c2_$L.log | grep -o '"value": [0-9.]*')"
  RIKI_LIB=$PWD/paper_2001_06770_b200/$L timeout 900 python bench.py --config 5 --steps 10 --warmup 3 --quick --no-cpu > gpurun_out/e19_c5_$L.log 2>&1
  echo "C5 $L: $(tail -c 1500 gpurun_out/e19_c5_$L.log | grep -o '"value": [0-9.]*')"
done
