# A/B: HEAD library (libriki_base.so) vs the atomics-counter + NVTX build; then C5 with the profiling pass
for L in libriki_base.so libriki.so libriki_base.so libriki.so; do
  RIKI_LIB=$PWD/paper_2001_06770_b200/$L timeout 900 python bench.py --config 5 --steps 4 --warmup 2 --quick --no-cpu > gpurun_out/e9_$L.log 2>&1
  echo "$L: $(tail -c 900 gpurun_out/e9_$L.log | grep -o '"value": [0-9.]*')"
done
timeout 1200 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu > gpurun_out/e9_c5_prof.log 2>&1
tail -c 2500 gpurun_out/e9_c5_prof.log
