timeout 600 python -m pytest tests/test_gpu_bake.py tests/test_gpu_parity.py -x -q -k "bake" > gpurun_out/gpu_tests28.log 2>&1; echo "pytest exit $?"
tail -1 gpurun_out/gpu_tests28.log
timeout 600 python bench.py --no-cpu --no-sweep --steps 5 > gpurun_out/bench28.json 2> gpurun_out/bench28.err; echo "bench exit $?"
python -c "import json; d=json.load(open('gpurun_out/bench28.json')); print(d['value'], json.dumps(d['splat']['roofline']), d['splat']['ms_per_step'])"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:bake -c 4 --csv --log-file gpurun_out/bake28.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-sweep > /dev/null 2>&1
grep -v "^==" gpurun_out/bake28.csv | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
ki,mi,vi=h.index('Kernel Name'),h.index('Metric Name'),h.index('Metric Value')
for x in r[1:]: print(x[ki][:30], x[mi], x[vi])
"
