# load-instruction variants vs DRAM bytes per random access (8 GiB working set)
export PATH=/usr/local/cuda/bin:$PATH
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o gpurun_out/randbench tools/randbench.cu
./gpurun_out/randbench > gpurun_out/e8_variants.jsonl 2>&1; cat gpurun_out/e8_variants.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex.sum,lts__t_requests_srcunit_tex.sum \
  --clock-control none --csv --log-file gpurun_out/e8_ncu.csv ./gpurun_out/randbench > /dev/null 2>&1
rm -f gpurun_out/randbench
