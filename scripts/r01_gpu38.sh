timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests38.log 2>&1; echo "pytest exit $?"
tail -1 gpurun_out/gpu_tests38.log
timeout 600 python bench.py --no-cpu --no-splat --no-sweep --steps 10 > gpurun_out/bench38.json 2> gpurun_out/bench38.err; echo "bench exit $?"
python -c "import json; d=json.load(open('gpurun_out/bench38.json')); print(d['value'], d['stages_ms'])"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"raster|delaunay" -c 4 --csv --log-file gpurun_out/geo.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-splat --no-sweep > /dev/null 2>&1
grep "raster\|delaunay" gpurun_out/geo.csv | awk -F'","' '{print $5, $NF}' | cut -c1-40,100-
