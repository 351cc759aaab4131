# Delaunay launch times under each value of a switch: bash scripts/dl_ab.sh TS_DL_MATCH 1 0
V=$1; shift
for X in "$@"; do
env $V=$X timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:delaunay -c 3 --csv --log-file gpurun_out/dl_$X.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-splat --no-sweep > /dev/null 2>&1
echo "$V=$X" $(grep -o '"gpu__time_duration.sum","[a-z]*","[0-9.,]*"' gpurun_out/dl_$X.csv | cut -d, -f3)
done
