# producer sweep: (producer warps, 32-byte loads in flight per thread)
for V in "12 4" "12 6" "14 4" "10 6"; do
set -- $V
sed -i "s/#define TS_H2_PRODW [0-9]*/#define TS_H2_PRODW $1/; s/constexpr int kIn8 = [0-9]*;/constexpr int kIn8 = $2;/" paper_2509_20198_b200/csrc/conv_tc2.cu
make -C paper_2509_20198_b200/csrc > /dev/null 2>&1 || echo build failed
timeout 600 python bench.py --no-cpu --no-splat --no-sweep --steps 10 > gpurun_out/b50.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/b50.json')); print('$V', d['value'], d['stages_ms']['cnn_refine'])"
done
