mkdir -p gpurun_out/prof
python bench.py --config 4a --steps 5 --warmup 3 > gpurun_out/prof/bench_config4a.json 2> gpurun_out/prof/bench_config4a.err; echo rc=$?
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_config4a.csv python bench.py --config 4a --steps 1 --warmup 3 --no-e2e --no-cpu --no-clocks > /dev/null 2>&1; echo ncu=$?
LM_NOPIV_TRACE=1 timeout 300 python tools/lu_trace.py 8192 2> gpurun_out/prof/lu8192_timeline_nopiv.txt; tail -2 gpurun_out/prof/lu8192_timeline_nopiv.txt
