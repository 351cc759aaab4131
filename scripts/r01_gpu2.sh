# bake rewrite + 3-product bf16x4: tests, precision, bench
timeout 600 python -m pytest tests/test_gpu_bake.py tests/test_gpu_tensorcore.py tests/test_gpu_parity.py -x -q > gpurun_out/gpu_tests2.log 2>&1; echo "pytest exit $?"
tail -15 gpurun_out/gpu_tests2.log
timeout 300 python scripts/precision_check.py 2>&1 | grep mode
timeout 600 python bench.py --no-cpu > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "bench exit $?"
cat gpurun_out/bench2.json; tail -3 gpurun_out/bench2.err
