timeout 600 python bench.py --no-cpu --no-splat --no-sweep --steps 10 > gpurun_out/bench39.json 2> gpurun_out/bench39.err; echo "bench exit $?"
tail -3 gpurun_out/bench39.err
python -c "import json; d=json.load(open('gpurun_out/bench39.json')); print(d['value'], d['stages_ms'], d['e2e'])"
