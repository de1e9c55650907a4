#!/bin/bash
# ncu evidence for one bench config: plain run first (must exit 0), then the
# launch list (gpu__time_duration per launch), then --set full on chosen kernels.
#   CONFIG=2 KERNELS='regex:trace_tiles|diag_scale_flat' bash tools/ncu_run.sh
set -u
C=${CONFIG:-2}
K=${KERNELS:-regex:.}
N=${NCAP:-3}
mkdir -p gpurun_out
CMD="python bench.py --config $C --steps 3 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/ncu_plain_c$C.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c$C.csv $CMD > gpurun_out/ncu_launch_c$C.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "$K" -c $N -o gpurun_out/prof_c$C -f $CMD > gpurun_out/ncu_full_c$C.log 2>&1
echo "rc=$?"
tail -3 gpurun_out/ncu_full_c$C.log
