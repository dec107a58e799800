#!/bin/bash
# per-kernel FP efficiency of one mid-build round (ncu, serialized) for library variants
for v in "$@"; do
  if [ "$v" = default ]; then lib=""; else lib=paper_2510_02774_b200/_build/variants/$v/libgrnnd_b200.so; fi
  GRNND_B200_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum,sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none -k regex:"pairs|decide|propagate" -s 100 -c 5 --csv --log-file gpurun_out/metrics_$v.csv python tools/prof_rounds.py 1000000 128 2 15 > /dev/null 2>&1
  echo "== $v"; python tools/metrics_summary.py gpurun_out/metrics_$v.csv
done
