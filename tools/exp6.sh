# random-access ceiling microbenchmark (tools/randbench.cu): timed run, then DRAM bytes per access under ncu
export PATH=/usr/local/cuda/bin:$PATH
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o gpurun_out/randbench tools/randbench.cu
./gpurun_out/randbench > gpurun_out/e6_randbench.jsonl 2>&1 && cat gpurun_out/e6_randbench.jsonl && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_requests_srcunit_tex.sum,lts__t_sectors_srcunit_tex.sum \
  --clock-control none --csv --log-file gpurun_out/e6_randbench_ncu.csv ./gpurun_out/randbench > gpurun_out/e6_ncu.log 2>&1
rm -f gpurun_out/randbench
echo done
