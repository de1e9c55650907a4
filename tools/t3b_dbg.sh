python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm_normwise" 2>&1 | tail -25
timeout 300 python bench.py --config 3b --steps 5 --warmup 2 --no-e2e --no-cpu 2>&1 | tail -12 | cut -c1-600
