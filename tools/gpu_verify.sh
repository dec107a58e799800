#!/bin/bash
# full gpu suite + smoke + C2 and C3 bench lines (a default-changing commit's check)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-verify}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_c2_bench.log 2>&1
timeout 1200 python bench.py --config c3 --no-cpu --steps 2 --warmup 3 > gpurun_out/${TAG}_c3_bench.log 2>&1
timeout 900 python bench.py --config c2c --no-cpu --steps 3 --warmup 3 > gpurun_out/${TAG}_c2c_bench.log 2>&1
