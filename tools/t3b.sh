# config 3b: split-K count A/B for Y.Z (LM_GEMM_SPLITS) and the resulting step
for sp in 0 16 25 37 50 74; do
  LM_GEMM_SPLITS=$sp timeout 300 python bench.py --config 3b --steps 20 --warmup 5 --no-e2e --no-cpu 2>/dev/null | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('3b splits=$sp', round(d['ms_per_step']*1e3,1),'us/step', r['kernel'], round(r['achieved'],2), round(r['ms_per_launch']*1e3,1), 'us', d.get('verified'))"
done
