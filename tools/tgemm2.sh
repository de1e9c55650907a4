set -u
for c in 3c 3b; do
  for st in 3 4 5 6; do
    LM_GEMM_TMA_ST=$st timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$c st=$st', round(d['ms_per_step']*1e3,1),'us/step', r['kernel'], round(r['achieved'],2), r['unit'], round(r['frac'],3))"
  done
  LM_GEMM_TMA=0 timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$c cp.async', round(d['ms_per_step']*1e3,1),'us/step', r['kernel'], round(r['achieved'],2), r['unit'], round(r['frac'],3))"
done
