for m in 0 32 128; do echo "tm exp $m"; LM_5A_EXP=$m timeout 60 python tools/power_probe.py 128 40000; done
