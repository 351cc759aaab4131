timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests37.log 2>&1; echo "pytest exit $?"
tail -1 gpurun_out/gpu_tests37.log
timeout 300 python scripts/precision_check.py 2>&1 | grep "mode [4]"
timeout 600 python bench.py --no-cpu --no-splat --no-sweep --steps 10 > gpurun_out/bench37.json 2> gpurun_out/bench37.err; echo "bench exit $?"
python -c "import json; d=json.load(open('gpurun_out/bench37.json')); print(d['value'], d['stages_ms'])"
source <(sed -n '/^run()/,/^}/p' scripts/r01_gpu15.sh)
run "0" v8
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"conv_tc_kernel|enc0" -c 6 --csv --log-file gpurun_out/merge.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-splat --no-sweep > /dev/null 2>&1
grep "conv_tc_kernel\|enc0" gpurun_out/merge.csv | awk -F'","' '{print $5, $NF}' | cut -c1-20,60-
