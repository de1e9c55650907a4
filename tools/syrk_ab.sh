timeout 300 python bench.py --config 3c --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('3c', round(d['ms_per_step']*1e3,1),'us/step', round(r['achieved'],2), round(r['frac'],3))"
