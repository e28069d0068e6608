# C5: expansion + apply kernels only, VF off vs on (plain launches)
export PATH=/usr/local/cuda/bin:$PATH
export RIKI_NO_GRAPHS=1
for VF in 1 0; do
RIKI_VF=$VF timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none \
    -k regex:"k_expand|k_vf_apply" -c 1200 --csv --log-file gpurun_out/e4_vf${VF}_c5.csv python bench.py --config 5 --steps 1 --warmup 1 --quick --no-cpu > gpurun_out/e4_vf${VF}.log 2>&1
done
echo done
