timeout 900 python -m pytest tests/test_gpu_country.py -x -q > gpurun_out/ct.log 2>&1; tail -3 gpurun_out/ct.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-splat --no-sweep --lazdec-tiles 0 --files 0 --sched-patches 0 > gpurun_out/bc.json 2> gpurun_out/bc.err; python -c "import json; d=json.load(open('gpurun_out/bc.json')); print(d['value'], d['country'])"
