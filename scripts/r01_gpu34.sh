timeout 600 python bench.py --no-cpu --no-splat --no-sweep --steps 10 > gpurun_out/bench34.json 2> gpurun_out/bench34.err; echo "bench exit $?"
python -c "import json; d=json.load(open('gpurun_out/bench34.json')); print(d['value'], d['stages_ms'])"
source <(sed -n '/^run()/,/^}/p' scripts/r01_gpu15.sh)
run "0" pf
timeout 600 python -m pytest tests/test_gpu_tensorcore.py -x -q 2>&1 | tail -1
