timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "chain or gemm" 2>&1 | tail -2
