timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests47.log 2>&1; echo "pytest exit $?"
tail -1 gpurun_out/gpu_tests47.log
timeout 300 python scripts/precision_check.py 2>&1 | grep "mode"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --no-cpu --no-splat --no-sweep --steps 10 > gpurun_out/bench47.json 2> gpurun_out/bench47.err; echo "bench exit $?"
python -c "import json; d=json.load(open('gpurun_out/bench47.json')); print(d['value'], d['stages_ms'], d['e2e']['value'])"
