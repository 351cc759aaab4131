# GPU tests + a 10-step bench (no CPU leg, no splat, no sweep) + halo2 launch times
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/q_tests.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/q_tests.log
timeout 600 python bench.py --no-cpu --no-splat --no-sweep --steps 10 > gpurun_out/q.json 2> gpurun_out/q.err; echo "bench exit $?"
python -c "import json; d=json.load(open('gpurun_out/q.json')); print(d['value'], d['stages_ms'], d['e2e']['value'])"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 100 -c 60 --csv --log-file gpurun_out/q_launch.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-splat --no-sweep > /dev/null 2>&1
python scripts/summarize_launches.py gpurun_out/q_launch.csv 2>/dev/null | head -20
