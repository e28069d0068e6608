set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py --config 5 --steps 3 --warmup 2 --quick --no-cpu > gpurun_out/e1_c5_default.log 2>&1
timeout 900 python bench.py --config 5 --steps 3 --warmup 2 --quick --no-cpu --vp > gpurun_out/e1_c5_vp.log 2>&1
timeout 600 python bench.py --config 2 --steps 5 --warmup 2 --quick --no-cpu --vp > gpurun_out/e1_c2_vp.log 2>&1
tail -c 600 gpurun_out/e1_*.log
