#!/bin/bash
# Run on the GPU box:  tools/profile_round.sh r01
# 1) launch list of one bench step (device time of every launch, cold-cache, serialised)
# 2) DRAM bytes of every expansion launch of one step (the bench's "traffic")
# 3) ncu --set full of the largest expansion launch (marginal flood level)
set -e
R=${1:-r01}
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/${R}_launches.csv python bench.py --steps 1 --warmup 1 --quick > gpurun_out/${R}_list.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
    --clock-control none -k regex:k_expand --csv --log-file gpurun_out/${R}_expand_dram.csv \
    python bench.py --steps 1 --warmup 1 --quick > gpurun_out/${R}_dram.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k k_expand -s 17 -c 1 \
    -o gpurun_out/${R}_expand_full python bench.py --steps 1 --warmup 1 --quick > gpurun_out/${R}_full.log 2>&1
echo profile_done
