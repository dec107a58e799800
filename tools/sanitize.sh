#!/bin/bash
# compute-sanitizer passes over a small build (tools/sanitize.py); logs to gpurun_out/<tag>_san_*.log
cd "$(dirname "$0")/.."
TAG=${1:-r2}
mkdir -p gpurun_out
export GRNND_EXACT_FIRST_ROUNDS=0
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
     python tools/sanitize.py 2000 > gpurun_out/${TAG}_san_${tool}.log 2>&1
  echo "rc=$?" >> gpurun_out/${TAG}_san_${tool}.log
done
