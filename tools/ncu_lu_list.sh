#!/bin/bash
set -u
mkdir -p gpurun_out
CMD="python tools/lu_once.py ${N:-8192}"
$CMD > gpurun_out/lu_once_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_lu.csv $CMD > gpurun_out/ncu_lu_list.log 2>&1
echo rc=$?
