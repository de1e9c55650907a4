#!/bin/bash
# ncu source-level capture of the pivot-free batched LU at one CTA per SM
set -u
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:lu_batched_nopiv -c 1 -o gpurun_out/ncu4b_small -f \
    python tools/lu4b_trace.py 148 > gpurun_out/ncu4b_small.log 2>&1
ncu -i gpurun_out/ncu4b_small.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu4b_small_sass.csv 2>/dev/null
echo done
