#!/bin/bash
# A/B of library variants (tools/variants.sh) on the GPU box: tools/ab.sh over $VARIANTS, twice
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-ab}
for rep in 1 2; do bash tools/ab.sh ${VARIANTS:-default} >> gpurun_out/${TAG}_ab.txt 2>&1; done
