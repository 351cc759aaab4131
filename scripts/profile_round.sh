# round-end evidence: per-launch time + DRAM bytes + tensor-pipe share for one
# bench step (after warm-up), one full ncu capture of the largest conv layer,
# and the bench line itself.
set -x
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -s 130 -c 200 --csv --log-file gpurun_out/r01_launch_metrics.csv python bench.py --steps 1 --warmup 3 --no-cpu --splat-points 20000000 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc_halo -s 9 -c 1 -o gpurun_out/r01_fuse0 python bench.py --steps 1 --warmup 1 --no-cpu --no-splat > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:bake_splat -s 1 -c 1 -o gpurun_out/r01_bake python bench.py --steps 1 --warmup 1 --no-cpu --splat-points 200000000 > /dev/null 2>&1
python bench.py > gpurun_out/r01_bench.json 2> gpurun_out/r01_bench.err
cat gpurun_out/r01_bench.json
