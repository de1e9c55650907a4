timeout 300 python bench.py --config 3a --steps 20 --warmup 5 --no-e2e --no-cpu 2>/dev/null | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('3a', round(d['ms_per_step']*1e3,1),'us/step', round(r['achieved'],1), r['unit'], round(r['frac'],3), d.get('verified'))"
