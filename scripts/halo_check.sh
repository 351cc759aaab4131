timeout 300 python -m pytest tests/test_gpu_tensorcore.py -q --tb=line 2>&1 | grep -E "Assert|passed|failed" | head -12
timeout 300 python bench.py --steps 5 --warmup 3 --precision 4 --no-cpu --no-splat > gpurun_out/bench_h3.json 2>gpurun_out/bench_h3.err; python -c "import json; d=json.load(open('gpurun_out/bench_h3.json')); print(d['value'], d['stages_ms'], d['roofline']['achieved'])" || tail -3 gpurun_out/bench_h3.err
bash scripts/launches.sh 4
