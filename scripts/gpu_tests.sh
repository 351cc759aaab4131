# the GPU test suite (as the driver runs it) + smoke
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?"
tail -15 gpurun_out/gpu_tests.log | grep -v Warning
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
