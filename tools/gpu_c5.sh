#!/bin/bash
# sharded GPU tests + the C5 one-rank probe (tools/c5_rank_probe.py), outputs under gpurun_out/${TAG}_*
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-c5}
timeout 900 python -m pytest tests/test_sharded.py -x -q > gpurun_out/${TAG}_pytest_sharded.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest_sharded.log
timeout 300 python tools/c5_rank_probe.py --n 4000000 > gpurun_out/${TAG}_probe_small.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_probe_small.log
timeout 900 python tools/c5_rank_probe.py > gpurun_out/${TAG}_probe_c5.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_probe_c5.log
timeout 900 python tools/c5_rank_probe.py --metric ip > gpurun_out/${TAG}_probe_c5_ip.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_probe_c5_ip.log
nvidia-smi --query-gpu=memory.total --format=csv >> gpurun_out/${TAG}_probe_c5.log
