# full GPU test suite + smoke on the current build
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02t_gpu_tests.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/r02t_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02t_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r02t_smoke.log
