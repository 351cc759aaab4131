# ncu launch times of one kernel (regex) in a bench step: bash scripts/k_time.sh raster_kernel
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:$1 -c 3 --csv --log-file gpurun_out/kt.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-splat --no-sweep > /dev/null 2>&1
echo "$1" $(grep -o '"gpu__time_duration.sum","[a-z]*","[0-9.,]*"' gpurun_out/kt.csv | cut -d, -f3)
