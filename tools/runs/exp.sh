timeout 300 python tools/host_overhead_probe.py 2>&1 | head -60
