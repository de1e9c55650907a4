#!/bin/bash
# Round evidence on the GPU box: per-config bench line, ncu launch list,
# DRAM traffic per roofline thunk, and one `ncu --set full` capture of each
# config's top kernel.  Output under gpurun_out/prof/ (copied to profiles/rNN
# afterwards).  Usage: CONFIGS="2 1 3a" bash tools/refresh_profiles.sh
set -u
O=gpurun_out/prof
mkdir -p $O
CONFIGS=${CONFIGS:-"2 1 3a 3b 3c 4a 4b 5a 5a-f32 5b"}
for C in $CONFIGS; do
  echo "== config $C"
  STEPS=20; [ "$C" = "4a" ] && STEPS=5; [ "$C" = "5a" ] && STEPS=5; [ "$C" = "5a-f32" ] && STEPS=5
  python bench.py --config $C --steps $STEPS --warmup 3 > $O/bench_config$C.json 2> $O/bench_config$C.err || { echo "bench $C failed"; tail -3 $O/bench_config$C.err; continue; }
  NL=1; ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_config$C.csv \
      python bench.py --config $C --steps $NL --warmup 3 --no-e2e --no-cpu --no-clocks > /dev/null 2>&1 || echo "launch list $C failed"
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
      --log-file $O/traffic_c$C.csv python tools/ncu_traffic.py run $C $O/traffic_c$C.order.json > /dev/null 2>&1 || echo "traffic $C failed"
done
echo done
