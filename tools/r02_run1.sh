set -x
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; free -g >> gpurun_out/host.txt; lscpu | head -20 >> gpurun_out/host.txt
timeout 900 python -m pytest tests/test_gpu_datagen.py tests/test_gpu_fullsize.py tests/test_gpu_batch.py tests/test_gpu_variants.py -q -x -m "gpu and not slow" > gpurun_out/t1.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/t1.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/b5a.json 2> gpurun_out/b5a.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/b5a.json; tail -20 gpurun_out/b5a.err
