bash tools/runs/exp.sh 2>&1 | grep CHAIN
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "chain" 2>&1 | tail -2
timeout 600 python bench.py --config 3b --steps 20 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['verified'], d['gpu_launches'])"
