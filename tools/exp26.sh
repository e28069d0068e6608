timeout 1500 python bench.py --config 5 --steps 10 --warmup 3 > gpurun_out/r02v_bench_c5.log 2>&1; echo "c5 rc=$?"
tail -c 4000 gpurun_out/r02v_bench_c5.log | grep -o '"value": [0-9.]*\|"latency_ms": {[^}]*}\|"parity": {"checked": [0-9]*, "identical": [0-9]*' | head -4
