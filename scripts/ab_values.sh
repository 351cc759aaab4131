# GPU tests, then the bench for each value of an execution switch:
#   bash scripts/ab_values.sh TS_ENC0 1 0
V=$1; shift
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/ab_tests.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/ab_tests.log
for X in "$@"; do
env $V=$X timeout 600 python bench.py --no-cpu --no-splat --no-sweep --steps 10 > gpurun_out/ab.json 2> gpurun_out/ab.err; echo "bench exit $?"
python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$V=$X', d['value'], d['stages_ms'], d['e2e']['value'])"
done
