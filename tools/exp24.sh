# large-graph variant only for batches of >= 8 queries in flight: config-5 bench line (latency p50/p99, throughput, parity gate)
timeout 1500 python bench.py --config 5 --steps 10 --warmup 3 > gpurun_out/r02t_bench_c5.log 2>&1; echo "c5 rc=$?"
tail -c 4000 gpurun_out/r02t_bench_c5.log | grep -o '"value": [0-9.]*\|"latency_ms": {[^}]*}\|"parity": {"checked": [0-9]*, "identical": [0-9]*' | head -4
timeout 900 python -m pytest tests/test_gpu_wikidata_scale.py -q -x -p no:cacheprovider > gpurun_out/r02t_tests.log 2>&1; tail -1 gpurun_out/r02t_tests.log
