# config 3b: skinny kernels (gemm_skinny.cu) on/off, plus the gemm parity tests
python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm" 2>&1 | tail -3
for sk in 1 0 1 0; do
  LM_GEMM_SKINNY=$sk timeout 300 python bench.py --config 3b --steps 50 --warmup 5 --no-e2e --no-cpu 2>/dev/null | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('3b skinny=$sk', round(d['ms_per_step']*1e3,2),'us/step', r['kernel'], round(r['achieved'],2), round(r['ms_per_launch']*1e3,2), 'us', d.get('verified'))"
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l3b.csv python bench.py --config 3b --steps 1 --warmup 3 --no-e2e --no-cpu --no-clocks > /dev/null 2>&1
python3 - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/l3b.csv')) if len(r)>10 and r[0].isdigit()]
for r in rows[-12:]: print(r[4][:60], r[7], r[8], r[-1])
PY
