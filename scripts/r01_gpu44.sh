timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "large_patches or random_patches" 2>&1 | tail -3
