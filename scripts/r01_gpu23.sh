timeout 900 python -m pytest tests/test_gpu_tensorcore.py tests/test_gpu_parity.py -x -q > gpurun_out/gpu_tests23.log 2>&1; echo "pytest exit $?"
tail -1 gpurun_out/gpu_tests23.log
timeout 300 python scripts/precision_check.py 2>&1 | grep "mode [234]"
timeout 600 python bench.py --no-cpu --no-splat --steps 5 > gpurun_out/bench23.json 2> gpurun_out/bench23.err; echo "bench exit $?"
python -c "import json; d=json.load(open('gpurun_out/bench23.json')); print(d['value'], d['stages_ms'], d['gpu_launches'])"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -s 100 -c 200 --csv --log-file gpurun_out/launch_metrics23.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-splat > /dev/null 2>&1; echo "ncu exit $?"
