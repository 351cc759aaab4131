timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests43.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/gpu_tests43.log
timeout 600 python bench.py --no-cpu --no-splat --no-sweep --steps 10 > gpurun_out/bench43.json 2> gpurun_out/bench43.err; echo "bench exit $?"
python -c "import json; d=json.load(open('gpurun_out/bench43.json')); print(d['value'], d['stages_ms'], d['e2e']['value'])"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"delaunay" -c 6 --csv --log-file gpurun_out/geo43.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-splat --no-sweep > /dev/null 2>&1
python - <<'PY'
import csv
r=list(csv.reader(open('gpurun_out/geo43.csv')))
hi=next(i for i,x in enumerate(r) if 'Metric Value' in x); h=r[hi]
for x in r[hi+1:]: print(x[h.index('Kernel Name')][:28], x[h.index('Metric Value')])
PY
