# CNN check after a kernel change: tensor-core tests, precision, timing, layer table
timeout 900 python -m pytest tests/test_gpu_tensorcore.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -4
timeout 300 python scripts/precision_check.py 0 5 2>&1 | tail -6
timeout 300 python scripts/cnn_time.py 5 4 2>&1 | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/layers_m5.csv python scripts/cnn_once.py 5 > /dev/null 2>&1
python scripts/layer_table.py gpurun_out/layers_m5.csv
