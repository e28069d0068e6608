timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02w_gpu_tests.log 2>&1
echo "pytest rc=$?"; tail -1 gpurun_out/r02w_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02w_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02w_smoke.log
