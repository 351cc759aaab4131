timeout 900 python -m pytest tests/test_gpu_tensorcore.py tests/test_gpu_parity.py -x -q > gpurun_out/gpu_tests19.log 2>&1; echo "pytest exit $?"
tail -1 gpurun_out/gpu_tests19.log
timeout 300 python scripts/precision_check.py 2>&1 | grep "mode [234]"
timeout 600 python bench.py --no-cpu --no-splat --steps 5 > gpurun_out/bench19.json 2> gpurun_out/bench19.err; echo "bench exit $?"
python -c "import json; d=json.load(open('gpurun_out/bench19.json')); print(d['value'], d['stages_ms'], d['gpu_launches'])"
source <(sed -n '/^run()/,/^}/p' scripts/r01_gpu15.sh)
run "0" x
