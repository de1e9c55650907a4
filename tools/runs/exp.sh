timeout 300 python tools/panel_probe.py 8192
timeout 300 python tools/panel_probe.py 4096
