# VF relaxation: parity tests, then quick A/B (RIKI_VF=0 / 1) at configs 5 and 2
timeout 900 python -m pytest tests/test_gpu_visited_fields.py -x -q > gpurun_out/e2_vf_tests.log 2>&1
tail -5 gpurun_out/e2_vf_tests.log
for C in 5 2; do
 for VF in 0 1; do
  RIKI_VF=$VF timeout 900 python bench.py --config $C --steps 3 --warmup 2 --quick --no-cpu > gpurun_out/e2_c${C}_vf${VF}.log 2>&1
  echo "C$C VF$VF: $(tail -c 700 gpurun_out/e2_c${C}_vf${VF}.log | grep -o '"value": [0-9.]*\|"section_ms": \[[^]]*\]' | tr '\n' ' ')"
 done
done
