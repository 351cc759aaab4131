# bake v2 tests + bench; ncu full of fuse.0/fuse.1 (halo2) and the bake kernel
timeout 600 python -m pytest tests/test_gpu_bake.py tests/test_gpu_parity.py -x -q -k "bake" > gpurun_out/gpu_tests3.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/gpu_tests3.log
timeout 600 python bench.py --no-cpu --steps 5 > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo "bench exit $?"
python -c "import json; d=json.load(open('gpurun_out/bench3.json')); print(d['value'], d['stages_ms'], json.dumps(d['splat']))"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc_halo2 -s 14 -c 2 -o gpurun_out/r01_halo2_fuse python bench.py --steps 1 --warmup 1 --no-cpu --no-splat > /dev/null 2>&1; echo "ncu1 exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bake_splat -s 1 -c 1 -o gpurun_out/r01_bake python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1; echo "ncu2 exit $?"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:bake -c 10 --csv --log-file gpurun_out/bake_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1; echo "ncu3 exit $?"
