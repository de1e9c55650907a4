for i in 1 2; do timeout 300 python tools/lu_trace.py 8192 2>&1 | grep -E "lu_factor" | tail -1; done
