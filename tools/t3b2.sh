for v in 1 0; do
  LM_GEMM_WIDE=$v timeout 300 python bench.py --config 3b --steps 20 --warmup 5 --no-e2e --no-cpu 2>/dev/null | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('3b wide=$v', round(d['ms_per_step']*1e3,1),'us/step', r['kernel'], round(r['achieved'],2), round(r['ms_per_launch']*1e3,1), 'us', d.get('verified'))"
done
timeout 300 python bench.py --config 3c --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('3c', round(d['ms_per_step']*1e3,1),'us/step', round(r['achieved'],2), round(r['frac'],3))"
timeout 600 python -m pytest -q -x tests/test_gpu_kernels.py tests/test_gpu_variants.py -k "gemm or syrk or chain" -p no:cacheprovider 2>&1 | tail -1
