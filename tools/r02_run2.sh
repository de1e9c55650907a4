mkdir -p gpurun_out/prof
python tools/prof_5a.py 128 20000
/usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:atb_schur -c 1 -o gpurun_out/prof/r02_5a128 -f python tools/prof_5a.py 128 20000 > gpurun_out/prof/r02_5a128.log 2>&1
echo ncu rc=$?
bash tools/sanitize.sh gpurun_out/sanitize
