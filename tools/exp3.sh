# per-kernel device time / DRAM / L2 hit rate of one C2 step, VF off vs on (plain launches)
export PATH=/usr/local/cuda/bin:$PATH
export RIKI_NO_GRAPHS=1
for VF in 0 1; do
RIKI_VF=$VF timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_requests_srcunit_tex_op_atom.sum,lts__t_sectors_srcunit_tex_op_atom.sum --clock-control none \
    -c 3000 --csv --log-file gpurun_out/e3_vf${VF}_c2.csv python bench.py --config 2 --steps 1 --warmup 1 --quick --no-cpu > gpurun_out/e3_vf${VF}.log 2>&1
done
timeout 600 python -m pytest tests/test_gpu_visited_fields.py -x -q -k "heavy" > gpurun_out/e3_heavy.log 2>&1
RIKI_VF=0 timeout 600 python -m pytest tests/test_gpu_visited_fields.py -x -q -k "heavy" > gpurun_out/e3_heavy_vf0.log 2>&1
echo done
