# final build (large-graph expansion at 4 blocks/SM): parity on every config, bench lines
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02s_gpu_tests.log 2>&1
echo "pytest rc=$?"; tail -1 gpurun_out/r02s_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02s_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02s_smoke.log
timeout 1500 python bench.py --config 5 --steps 10 --warmup 3 > gpurun_out/r02s_bench_c5.log 2>&1; echo "c5 rc=$?"
timeout 900 python bench.py --config 2 --steps 20 --warmup 5 > gpurun_out/r02s_bench_c2.log 2>&1; echo "c2 rc=$?"
timeout 1500 python bench.py --config 3 --steps 5 --warmup 3 --cpu-sample 16 > gpurun_out/r02s_bench_c3.log 2>&1; echo "c3 rc=$?"
timeout 1800 python bench.py --config 4 --steps 5 --warmup 3 --cpu-sample 16 > gpurun_out/r02s_bench_c4.log 2>&1; echo "c4 rc=$?"
