timeout 900 python -m pytest tests/test_gpu_tensorcore.py tests/test_gpu_parity.py -x -q > gpurun_out/gpu_tests12.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/gpu_tests12.log
timeout 300 python scripts/precision_check.py 2>&1 | grep "mode [234]"
timeout 600 python bench.py --no-cpu --no-splat --steps 5 > gpurun_out/bench12.json 2> gpurun_out/bench12.err; echo "bench exit $?"
python -c "import json; d=json.load(open('gpurun_out/bench12.json')); print(d['value'], d['stages_ms'], d['gpu_launches'])"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:conv_tc_halo2 -s 34 -c 34 --csv --log-file gpurun_out/h2_12.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-splat > /dev/null 2>&1
python - <<PY
import csv
r=list(csv.reader(open('gpurun_out/h2_12.csv')))
hi=next(i for i,x in enumerate(r) if 'Metric Value' in x); h=r[hi]; vi=h.index('Metric Value')
v=[float(x[vi].replace(',',''))/1e3 for x in r[hi+1:]]
print(' '.join(f'{t:.0f}' for t in v), ' total', round(sum(v)))
PY
