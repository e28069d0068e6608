# atomic read (atomicOr 0) vs load before the dependent atomicAnd: time and DRAM bytes per access
export PATH=/usr/local/cuda/bin:$PATH
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o gpurun_out/randbench tools/randbench.cu
./gpurun_out/randbench > gpurun_out/e11_variants.jsonl 2>&1; cat gpurun_out/e11_variants.jsonl | grep -v '"working_set_mib": 64,'
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex.sum,lts__t_requests_srcunit_tex.sum \
  --clock-control none --csv --log-file gpurun_out/e11_ncu.csv ./gpurun_out/randbench > /dev/null 2>&1
rm -f gpurun_out/randbench
