timeout 120 python tools/pcie_probe.py 2>&1 | tail -4
for i in 1 2; do timeout 300 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2 e2e', d['e2e']['value'], d['e2e']['ms_per_step'])"; done
timeout 300 python bench.py --config 1 --steps 10 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1 e2e', d['e2e']['value'], d['e2e']['ms_per_step'])"
