#!/bin/bash
# per-kernel launch times of a short C2 schedule + one full ncu capture of round 21's pair-phase kernels
TAG=${1:-x}; REGEX=${2:-"pairs|decide"}; SKIP=${3:-100}; CNT=${4:-5}
cd "$(dirname "$0")/.."
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
   python tools/prof_rounds.py 1000000 128 2 15 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launch_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$REGEX" -s $SKIP -c $CNT \
   -o gpurun_out/${TAG}_full -f python tools/prof_rounds.py 1000000 128 2 15 > gpurun_out/${TAG}_ncu.log 2>&1
cat gpurun_out/${TAG}_launch_summary.txt
