timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -q -x -k "lu or config4a" 2>&1 | tail -2
