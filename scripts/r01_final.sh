timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_f.log 2>&1; echo "pytest exit $?"
tail -1 gpurun_out/gpu_tests_f.log
timeout 300 python scripts/precision_check.py 2>&1 | grep "mode"
for V in 1 0; do
TS_FINAL=$V timeout 600 python bench.py --no-cpu --no-splat --no-sweep --steps 10 > gpurun_out/bf.json 2> gpurun_out/bf.err; echo "bench exit $?"
python -c "import json; d=json.load(open('gpurun_out/bf.json')); print('final $V', d['value'], d['stages_ms'], d['e2e']['value'])"
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"conv_final" -c 2 --csv --log-file gpurun_out/fin.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-splat --no-sweep > /dev/null 2>&1
grep conv_final gpurun_out/fin.csv | awk -F'","' '{print $NF}'
