timeout 900 python -m pytest tests/test_gpu_tensorcore.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
timeout 300 python scripts/precision_check.py 5 2>&1 | grep "mode 5"
timeout 300 python scripts/cnn_time.py 5 2>&1 | tail -1
TS_LIB_PATH=build/prof/libts_b200.so timeout 300 python scripts/cnn_once.py 5 2>&1 | grep h2prof | tail -36 | sed 's/h2prof //' | cut -c1-200
