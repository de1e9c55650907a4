#!/bin/bash
# DRAM traffic per roofline thunk + one `ncu --set full` capture of the top
# kernel(s) of each config, into gpurun_out/prof/.  Run after
# tools/refresh_profiles.sh (each command below exited 0 there without ncu).
set -u
O=gpurun_out/prof
mkdir -p $O
declare -A K=( [1]="regex:lm_prog" [2]="regex:trace_tiles|diag_scale_cols32" [3a]="regex:gemv_cm32" \
               [3b]="regex:dgemm_tall|dgemm_dmma|splitk" [3c]="regex:dgemm_dmma" [4a]="regex:lu_panel_cluster|dgemm_dmma" \
               [4b]="regex:lu_batched_nopiv|lu_batched_shift|lu_batched_rows" [5a]="regex:atb_schur" [5a]="regex:atb_schur" [5a-f32]="regex:atb_schur" [5b]="regex:lm_prog|trace_quads" )
declare -A NC=( [1]=1 [2]=2 [3a]=1 [3b]=2 [3c]=1 [4a]=2 [4b]=2 [5a]=3 [5a-f32]=3 [5b]=2 )
for C in ${CONFIGS:-2 1 3a 3b 3c 4a 4b 5a 5a-f32 5b}; do
  echo "== config $C"
  if [ "$C" != "4a" ] && [ "$C" != "4b" ]; then
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
        --log-file $O/traffic_c$C.csv python tools/ncu_traffic.py run $C $O/traffic_c$C.order.json > /dev/null 2>&1 || echo "traffic $C failed"
  fi
  ncu --set full --clock-control none --import-source on -k "${K[$C]}" -c ${NC[$C]} -o $O/full_c$C -f \
      python bench.py --config $C --steps 1 --warmup 3 --no-e2e --no-cpu --no-clocks > $O/full_c$C.log 2>&1 || echo "full $C failed"
  python tools/ncu_summary.py $O/full_c$C.ncu-rep > $O/full_c$C.txt 2>&1
  # keep only the reports asked for (gpurun copies back <= 64 MiB)
  case " ${KEEP:-2} " in *" $C "*) ;; *) rm -f $O/full_c$C.ncu-rep ;; esac
done
echo done
