timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests52.log 2>&1; echo "pytest exit $?"
tail -1 gpurun_out/gpu_tests52.log
for V in 1 0; do
TS_BRANCH_STREAMS=$V timeout 600 python bench.py --no-cpu --no-splat --no-sweep --steps 10 > gpurun_out/bench52.json 2> gpurun_out/bench52.err; echo "bench exit $?"
python -c "import json; d=json.load(open('gpurun_out/bench52.json')); print('branches $V', d['value'], d['stages_ms'], d['e2e']['value'])"
done
