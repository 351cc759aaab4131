# raster occupancy variants: (launch-bound CTAs/SM, shared-memory point cache)
for V in "2 512" "3 512" "4 384"; do
set -- $V
sed -i "s/__launch_bounds__(kThreads, [0-9])/__launch_bounds__(kThreads, $1)/; s/constexpr int kSmemPts = [0-9]*;/constexpr int kSmemPts = $2;/" paper_2509_20198_b200/csrc/raster.cu
make -C paper_2509_20198_b200/csrc > /dev/null 2>&1 || echo build failed
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:raster -c 2 --csv --log-file gpurun_out/ras.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-splat --no-sweep > /dev/null 2>&1
echo "raster $V: $(grep raster gpurun_out/ras.csv | awk -F'","' '{print $NF}' | tr '\n' ' ')"
done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
