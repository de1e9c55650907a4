#!/bin/bash
# One gpurun call: probes, GPU tests, smoke, bench.  Logs land in gpurun_out/.
set -u
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
( timeout 60 ./build/fp64_probe > gpurun_out/fp64_probe.txt 2>&1 ) || echo "probe rc=$?" >> gpurun_out/fp64_probe.txt
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
for c in ${BENCH_CONFIGS:-2 1}; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
  echo "bench c$c rc=$?" >> gpurun_out/bench_c$c.err
done
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log; cat gpurun_out/bench_c*.json | cut -c1-400
