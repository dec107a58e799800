#!/bin/bash
# C1 and C4 bench lines (outputs gpurun_out/${TAG}_c{1,4}_bench.log)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-c14}
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 > gpurun_out/${TAG}_c1_bench.log 2>&1
timeout 1200 python bench.py --config c4 --no-cpu --steps 2 --warmup 3 > gpurun_out/${TAG}_c4_bench.log 2>&1
