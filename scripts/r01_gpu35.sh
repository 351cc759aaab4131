timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests35.log 2>&1; echo "pytest exit $?"
tail -1 gpurun_out/gpu_tests35.log
timeout 300 python scripts/precision_check.py 2>&1 | grep "mode [234]"
timeout 600 python bench.py --no-cpu --no-splat --no-sweep --steps 10 > gpurun_out/bench35.json 2> gpurun_out/bench35.err; echo "bench exit $?"
python -c "import json; d=json.load(open('gpurun_out/bench35.json')); print(d['value'], d['stages_ms'])"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:enc0 -c 3 --csv --log-file gpurun_out/enc0.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-splat --no-sweep > /dev/null 2>&1
grep enc0 gpurun_out/enc0.csv | awk -F'","' '{print $NF}'
