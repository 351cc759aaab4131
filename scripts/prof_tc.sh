timeout 300 python -m pytest tests/test_gpu_tensorcore.py -q --tb=line -k "3-shape0 or 3-shape2 or 3-shape6" 2>&1 | grep -E "Assert|passed|failed" | head
timeout 300 python bench.py --steps 3 --warmup 3 --precision 3 --no-cpu --no-splat 2>&1 | tail -5
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc -s 6 -c 3 -o gpurun_out/prof_tc python bench.py --steps 1 --warmup 1 --precision 2 --no-cpu --no-splat > /dev/null 2>&1
ls -la gpurun_out/
