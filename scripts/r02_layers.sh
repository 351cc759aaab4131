# per-launch time / DRAM / tensor-pipe of one CNN refine (1,024 tiles) per mode
for M in 5 4; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/layers_m$M.csv python scripts/cnn_once.py $M > /dev/null 2>&1
echo "mode $M rc $?"
done
timeout 300 python scripts/cnn_time.py 4 5 2
