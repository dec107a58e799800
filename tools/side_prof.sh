#!/bin/bash
# ncu --set full of the side kernels over rounds 1-6 of a C2-shape build; keeps CSV exports
# (raw metrics, details, decide/apply source pages) and drops the large .ncu-rep.
cd "$(dirname "$0")/.."
TAG=${1:-r2c}
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"decide_kernel|apply_round_kernel|bin_kernel|scatter_kernel|segsort_light|segsort_medium|segsort_heavy|count_targets" \
  -c ${CNT:-48} -o /tmp/${TAG}_side -f python tools/prof_rounds.py 1000000 128 1 6 > gpurun_out/${TAG}_ncu.log 2>&1
python tools/ncu_to_json.py /tmp/${TAG}_side.ncu-rep gpurun_out/${TAG}_side_ncu.json "side kernels, rounds 1-6 of a C2-shape build (T1=1 T2=6)" > /dev/null 2>&1
ncu -i /tmp/${TAG}_side.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>&1
for k in decide_kernel apply_round_kernel; do
  ncu -i /tmp/${TAG}_side.ncu-rep --page source --csv --print-source cuda -k regex:$k -c 1 -s ${SRCSKIP:-4} > gpurun_out/${TAG}_src_${k}.csv 2>&1
done
ls -la gpurun_out
