#!/bin/bash
# launch list (per-kernel device time) for one bench config; plain run first.
set -u
C=${CONFIG:-4a}
CMD="python bench.py --config $C --steps ${STEPS:-1} --warmup 3 --no-e2e --no-cpu"
mkdir -p gpurun_out
$CMD > gpurun_out/ncu_plain_c$C.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c$C.csv -c ${NLAUNCH:-20000} $CMD > gpurun_out/ncu_launch_c$C.log 2>&1
echo "rc=$?"
