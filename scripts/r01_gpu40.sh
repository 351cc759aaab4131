timeout 600 python -m pytest tests/test_gpu_bake.py tests/test_gpu_parity.py -x -q -k "bake" > gpurun_out/gpu_tests40.log 2>&1; echo "pytest exit $?"
tail -1 gpurun_out/gpu_tests40.log
timeout 600 python bench.py --no-cpu --no-sweep --steps 5 > gpurun_out/bench40.json 2> gpurun_out/bench40.err; echo "bench exit $?"
python -c "import json; d=json.load(open('gpurun_out/bench40.json')); print(d['value'], json.dumps(d['splat']['roofline']), d['splat']['ms_per_step'])"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:bake_splat -c 2 --csv --log-file gpurun_out/bake40.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-sweep > /dev/null 2>&1
grep bake_splat gpurun_out/bake40.csv | awk -F'","' '{print $NF}'
