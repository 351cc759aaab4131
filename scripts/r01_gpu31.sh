timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests31.log 2>&1; echo "pytest exit $?"
tail -1 gpurun_out/gpu_tests31.log
timeout 300 python scripts/precision_check.py 2>&1 | grep "mode [234]"
timeout 600 python bench.py --no-cpu --no-splat --no-sweep --steps 10 > gpurun_out/bench31.json 2> gpurun_out/bench31.err; echo "bench exit $?"
python -c "import json; d=json.load(open('gpurun_out/bench31.json')); print(d['value'], d['stages_ms'], d['e2e']['value'])"
