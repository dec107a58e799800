#!/bin/bash
# sharded-path GPU tests (gloo multi-process on one GPU + one-rank NCCL), outputs gpurun_out/${TAG}_*
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-sh}
timeout 1200 python -m pytest tests/test_sharded.py -m gpu -q > gpurun_out/${TAG}_pytest_sharded.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest_sharded.log
