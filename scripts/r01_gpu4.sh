# splat v3 (interior key lists) + producer in-flight sweep for halo2
timeout 600 python -m pytest tests/test_gpu_bake.py tests/test_gpu_parity.py -x -q -k "bake" > gpurun_out/gpu_tests4.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/gpu_tests4.log
timeout 600 python bench.py --no-cpu --steps 5 > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo "bench exit $?"
python -c "import json; d=json.load(open('gpurun_out/bench4.json')); print(d['value'], d['stages_ms'], json.dumps(d['splat']))"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:bake -c 4 --csv --log-file gpurun_out/bake_launches4.csv python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1; echo "ncu exit $?"
python scripts/summarize_launches.py gpurun_out/bake_launches4.csv
for K in 16 24; do
  sed -i "s/constexpr int kInflight = [0-9]*;/constexpr int kInflight = $K;/" paper_2509_20198_b200/csrc/conv_tc2.cu
  make -C paper_2509_20198_b200/csrc > /dev/null 2>&1 || echo "build failed $K"
  timeout 300 python bench.py --no-cpu --no-splat --steps 5 > gpurun_out/bench_k$K.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/bench_k$K.json')); print('kInflight $K', d['value'], d['stages_ms'])"
done
