timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests9.log 2>&1; echo "pytest exit $?"
tail -15 gpurun_out/gpu_tests9.log | grep -v Warn
timeout 300 python scripts/precision_check.py 2>&1 | grep mode
TS_POLY=0 timeout 300 python scripts/precision_check.py 2>&1 | grep "mode 4"
timeout 600 python bench.py --no-cpu --no-splat --steps 5 > gpurun_out/bench9.json 2> gpurun_out/bench9.err; echo "bench exit $?"
python -c "import json; d=json.load(open('gpurun_out/bench9.json')); print(d['value'], d['stages_ms'], d['gpu_launches'])"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -s 120 -c 200 --csv --log-file gpurun_out/launch_metrics9.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-splat > /dev/null 2>&1; echo "ncu exit $?"
