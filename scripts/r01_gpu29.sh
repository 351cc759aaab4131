for W in 8 12; do
sed -i "s/#define TS_H2_PRODW [0-9]*/#define TS_H2_PRODW $W/" paper_2509_20198_b200/csrc/conv_tc2.cu
make -C paper_2509_20198_b200/csrc > /dev/null 2>&1 || echo build failed
timeout 600 python bench.py --no-cpu --no-splat --no-sweep --steps 5 > gpurun_out/bench29.json 2> gpurun_out/bench29.err
python -c "import json; d=json.load(open('gpurun_out/bench29.json')); print('prodw $W', d['value'], d['stages_ms'])"
source <(sed -n '/^run()/,/^}/p' scripts/r01_gpu15.sh)
run "0" w$W
done
timeout 600 python -m pytest tests/test_gpu_tensorcore.py -x -q 2>&1 | tail -1
