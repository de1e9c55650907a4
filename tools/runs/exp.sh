timeout 1500 python -m pytest tests -q -x -m gpu 2>&1 | tail -4
timeout 600 python bench.py --config 5b --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-400
