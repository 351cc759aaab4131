P=${1:-3}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 120 -c 200 --csv --log-file gpurun_out/launches_p$P.csv python bench.py --steps 2 --warmup 3 --precision $P --no-cpu --no-splat > /dev/null 2>&1
wc -l gpurun_out/launches_p$P.csv
