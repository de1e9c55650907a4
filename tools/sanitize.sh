#!/bin/bash
# compute-sanitizer pass over the GPU tests that exercise the
# riskiest kernels: mbarrier/TMA/tcgen05 rings of the batched 5a kernels,
# the cluster LU panel (st.async mailboxes), the cooperative wavefront
# solve, the batched LU.  Usage: bash tools/sanitize.sh OUTDIR
out=${1:-gpurun_out/sanitize}
mkdir -p "$out"
CS=/usr/local/cuda/bin/compute-sanitizer
SEL_BATCH="tests/test_gpu_batch.py"
SEL_LU="tests/test_gpu_kernels.py -k lu_factor_bitwise_values_and_pivots or lu_factor_large_general_bitwise or lu_singular"
for tool in memcheck racecheck synccheck; do
  for sel in batch lu; do
    if [ $sel = batch ]; then args="$SEL_BATCH"; else args="$SEL_LU"; fi
    echo "== $tool $sel" | tee -a "$out/summary.txt"
    timeout 1500 $CS --tool $tool --error-exitcode 9 --print-limit 50 --log-file "$out/${tool}_${sel}.log" \
      python -m pytest $args -q -x -m gpu -p no:cacheprovider > "$out/${tool}_${sel}.pytest.log" 2>&1
    rc=$?
    echo "rc=$rc" | tee -a "$out/summary.txt"
    tail -3 "$out/${tool}_${sel}.pytest.log" | tee -a "$out/summary.txt"
    grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard|Error" "$out/${tool}_${sel}.log" | tail -5 | tee -a "$out/summary.txt"
  done
done
