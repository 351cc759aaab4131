for X in 2 4 8; do
TS_DL_ILP=$X timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:delaunay -c 3 --csv --log-file gpurun_out/dl_$X.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-splat --no-sweep > /dev/null 2>&1
echo "ILP $X"; grep -o '"gpu__time_duration.sum","[a-z]*","[0-9.,]*"' gpurun_out/dl_$X.csv
done
