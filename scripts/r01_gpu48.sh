timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests48.log 2>&1; echo "pytest exit $?"
tail -1 gpurun_out/gpu_tests48.log
