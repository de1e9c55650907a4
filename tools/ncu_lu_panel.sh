#!/bin/bash
set -u
mkdir -p gpurun_out
CMD="python tools/lu_probe.py 4096"
$CMD > gpurun_out/lu_probe_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"lu_panel_cluster|exact_update128|tri_cols" -s 20 -c 3 -o gpurun_out/prof_lu -f $CMD > gpurun_out/ncu_lu.log 2>&1
echo rc=$?
