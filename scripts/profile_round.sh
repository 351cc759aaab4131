# Round evidence (run under gpurun): per-launch time / DRAM / tensor-pipe of
# one bench step, the splat launches, full ncu captures of the top CNN kernel
# (fuse.0 on the wide-M halo kernel) and of the splat kernel, then the bench
# line itself.  Summaries are written by scripts/summarize_round.py.
set -x
R=${R:-r02}
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -s 100 -c 200 --csv --log-file gpurun_out/${R}_launch_metrics.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-splat --no-sweep --country-tiles 0 --lazdec-tiles 0 --files 0 --sched-patches 0 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:bake -c 4 --csv --log-file gpurun_out/${R}_bake_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-sweep --country-tiles 0 --lazdec-tiles 0 --files 0 --sched-patches 0 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc_halo2 -s 70 -c 1 -o gpurun_out/${R}_fuse0 python bench.py --steps 1 --warmup 1 --no-cpu --no-splat --no-sweep --country-tiles 0 --lazdec-tiles 0 --files 0 --sched-patches 0 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bake_splat -s 1 -c 1 -o gpurun_out/${R}_splat python bench.py --steps 1 --warmup 1 --no-cpu --no-sweep --country-tiles 0 --lazdec-tiles 0 --files 0 --sched-patches 0 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:raster_kernel -s 1 -c 1 -o gpurun_out/${R}_raster python bench.py --steps 1 --warmup 1 --no-cpu --no-splat --no-sweep --country-tiles 0 --lazdec-tiles 0 --files 0 --sched-patches 0 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:delaunay_kernel -s 1 -c 1 -o gpurun_out/${R}_delaunay python bench.py --steps 1 --warmup 1 --no-cpu --no-splat --no-sweep --country-tiles 0 --lazdec-tiles 0 --files 0 --sched-patches 0 > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err
cat gpurun_out/${R}_bench.json
# the reference arm as the driver runs it (timed, for the record)
T0=$(date +%s)
timeout 900 python bench.py --impl reference > gpurun_out/${R}_bench_ref.json 2> gpurun_out/${R}_bench_ref.err
echo "reference arm wall $(( $(date +%s) - T0 )) s"
cat gpurun_out/${R}_bench_ref.json
