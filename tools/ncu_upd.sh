#!/bin/bash
set -u
mkdir -p gpurun_out
CMD="python tools/lu_once.py 8192"
$CMD > gpurun_out/lu_once_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"exact_update128" -s 20 -c 2 -o gpurun_out/prof_upd -f $CMD > gpurun_out/ncu_upd.log 2>&1
echo rc=$?
