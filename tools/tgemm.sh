set -u
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_kernels.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py -p no:cacheprovider > gpurun_out/tgemm.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/tgemm.log
for c in 3b 3c 4a; do
  for v in 1 0; do
    LM_GEMM_TMA=$v timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$c tma=$v', round(d['ms_per_step']*1e3,1),'us/step', r['kernel'], round(r['achieved'],2), r['unit'], round(r['frac'],3), d.get('verified'))"
  done
done
