timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests36.log 2>&1; echo "pytest exit $?"
tail -1 gpurun_out/gpu_tests36.log
timeout 300 python scripts/precision_check.py 2>&1 | grep "mode [34]"
for V in 1 0; do
TS_TC_WIDE=$V timeout 600 python bench.py --no-cpu --no-splat --no-sweep --steps 10 > gpurun_out/bench36.json 2> gpurun_out/bench36.err; echo "bench exit $?"
python -c "import json; d=json.load(open('gpurun_out/bench36.json')); print('wide $V', d['value'], d['stages_ms'])"
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:conv_tc_kernel -c 4 --csv --log-file gpurun_out/merge.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-splat --no-sweep > /dev/null 2>&1
grep conv_tc_kernel gpurun_out/merge.csv | awk -F'","' '{print $NF}'
