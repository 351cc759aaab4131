timeout 900 python -m pytest tests/test_gpu_tensorcore.py tests/test_gpu_parity.py -x -q > gpurun_out/gpu_tests25.log 2>&1; echo "pytest exit $?"
tail -1 gpurun_out/gpu_tests25.log
timeout 300 python scripts/precision_check.py 2>&1 | grep "mode [234]"
for V in auto 1; do
if [ $V = auto ]; then unset TS_H2_STACK; else export TS_H2_STACK=$V; fi
timeout 600 python bench.py --no-cpu --no-splat --no-sweep --steps 5 > gpurun_out/bench25.json 2> gpurun_out/bench25.err; echo "bench exit $?"
python -c "import json; d=json.load(open('gpurun_out/bench25.json')); print('stack=$V', d['value'], d['stages_ms'], d['gpu_launches'])"
done
unset TS_H2_STACK
source <(sed -n '/^run()/,/^}/p' scripts/r01_gpu15.sh)
run "0" x
