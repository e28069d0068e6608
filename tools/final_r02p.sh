# final round-2 evidence of the current build: bench lines (configs 5 and 2), per-launch DRAM of one step per
# config (roofline.traffic), ncu full capture of the longest config-2 k_expand launch
export PATH=/usr/local/cuda/bin:$PATH
timeout 1500 python bench.py --config 5 --steps 10 --warmup 3 > gpurun_out/r02p_bench_c5.log 2>&1; echo "c5 rc=$?"
timeout 900 python bench.py --config 2 --steps 20 --warmup 5 > gpurun_out/r02p_bench_c2.log 2>&1; echo "c2 rc=$?"
FULL=0 timeout 1800 bash tools/profile_r02.sh r02p 5; echo "prof5 rc=$?"
timeout 1500 bash tools/profile_r02.sh r02p 2; echo "prof2 rc=$?"
ls gpurun_out | grep r02p
