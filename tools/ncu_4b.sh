#!/bin/bash
# ncu --set full of the config-4b batched LU kernel (variant from LM_BATCHED_LU)
set -u
mkdir -p gpurun_out
V=${LM_BATCHED_LU:-nopiv}
python tools/prof_4b.py > gpurun_out/prof4b_$V.txt 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:lu_batched -c 2 -o gpurun_out/ncu4b_$V -f \
    python tools/prof_4b.py > gpurun_out/ncu4b_$V.log 2>&1
ncu -i gpurun_out/ncu4b_$V.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu4b_${V}_sass.csv 2>/dev/null
cat gpurun_out/prof4b_$V.txt
