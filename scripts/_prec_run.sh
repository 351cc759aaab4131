python scripts/cnn_time.py 5
python scripts/precision_check.py 5
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/cnn_launch_m6b.csv python scripts/cnn_once.py 5 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv_tc_halo2 -s 32 -c 1 -o gpurun_out/fuse0_m6 python scripts/cnn_once.py 5 > /dev/null 2>&1
