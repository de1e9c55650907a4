timeout 300 python tools/small_lu_probe.py
