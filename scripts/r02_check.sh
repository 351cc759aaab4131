# full GPU suite + smoke + bench line
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?"
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['e2e']['value'], d['stages_ms'], d['roofline']['frac'], d['splat']['value'], d['clocks'])"
tail -3 gpurun_out/bench.err
