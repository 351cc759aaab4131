for k in raster_kernel delaunay_kernel conv_direct; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/prof_$k python bench.py --steps 1 --warmup 1 --no-cpu --no-splat > /dev/null 2>&1
done
ls gpurun_out/*.ncu-rep
