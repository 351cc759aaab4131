timeout 900 python -m pytest tests/test_gpu_tensorcore.py tests/test_gpu_parity.py -x -q > gpurun_out/gpu_tests24.log 2>&1; echo "pytest exit $?"
tail -1 gpurun_out/gpu_tests24.log
timeout 300 python scripts/precision_check.py 2>&1 | grep "mode [234]"
for V in 1 0; do
TS_H2_1X1=$V timeout 600 python bench.py --no-cpu --no-splat --no-sweep --steps 5 > gpurun_out/bench24.json 2> gpurun_out/bench24.err; echo "bench exit $?"
python -c "import json; d=json.load(open('gpurun_out/bench24.json')); print('1x1=$V', d['value'], d['stages_ms'], d['gpu_launches'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"delaunay|conv_tc|raster" -s 40 -c 60 --csv --log-file gpurun_out/l24.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-splat --no-sweep > /dev/null 2>&1
python scripts/summarize_launches.py gpurun_out/l24.csv
