timeout 600 python -m pytest tests/test_gpu_bake.py tests/test_gpu_parity.py -x -q -k "bake" > gpurun_out/gpu_tests8.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/gpu_tests8.log
timeout 600 python bench.py --no-cpu --steps 5 > gpurun_out/bench8.json 2> gpurun_out/bench8.err; echo "bench exit $?"
python -c "import json; d=json.load(open('gpurun_out/bench8.json')); print(d['value'], d['stages_ms'], json.dumps(d['splat']))"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bake_splat -s 1 -c 1 -o gpurun_out/r01_bake5 python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1; echo "ncu exit $?"
