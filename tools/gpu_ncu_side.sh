#!/bin/bash
# ncu --set full captures (source counters) of decide (rounds 3 and 16) and apply (round 16)
# of a C2-shape build; source pages exported as CSV.  Outputs gpurun_out/${TAG}_*
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-side}
for spec in "decide:2:r3" "decide:15:r16" "apply_round:16:r16"; do
  IFS=: read k s r <<< "$spec"
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s $s -c 1 \
     -o gpurun_out/${TAG}_${k}_${r} -f python tools/prof_rounds.py 1000000 128 2 15 > gpurun_out/${TAG}_${k}_${r}.log 2>&1
  ncu -i gpurun_out/${TAG}_${k}_${r}.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_${k}_${r}_sass.csv 2>/dev/null
  ncu -i gpurun_out/${TAG}_${k}_${r}.ncu-rep --page source --csv --print-source cuda > gpurun_out/${TAG}_${k}_${r}_cuda.csv 2>/dev/null
  ncu -i gpurun_out/${TAG}_${k}_${r}.ncu-rep --page raw --csv > gpurun_out/${TAG}_${k}_${r}_raw.csv 2>/dev/null
done
