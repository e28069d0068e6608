# L2 fetch granularity (cudaLimitMaxL2FetchGranularity) vs random-access throughput and DRAM bytes per access
export PATH=/usr/local/cuda/bin:$PATH
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o gpurun_out/randbench tools/randbench.cu
for G in 0 32 64 128; do echo "== gran $G"; ./gpurun_out/randbench $G; done > gpurun_out/e7_gran.jsonl 2>&1
cat gpurun_out/e7_gran.jsonl
for G in 32 128; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex.sum,lts__t_requests_srcunit_tex.sum \
  --clock-control none --csv --log-file gpurun_out/e7_ncu_g$G.csv ./gpurun_out/randbench $G > /dev/null 2>&1
done
rm -f gpurun_out/randbench
