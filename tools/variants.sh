#!/bin/bash
# Build A/B variants of libgrnnd_b200.so with compile-time knobs into _build/variants/<name>/.
# usage: tools/variants.sh name "-DKNOB=1 -DOTHER=2" [name2 "flags2" ...]
set -e
cd "$(dirname "$0")/../paper_2510_02774_b200/csrc"
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  out=../_build/variants/$name; mkdir -p $out/obj
  for f in capi propagate group apply reverse search; do
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
      -Xcompiler -fPIC,-O2 -I../../include -I. --expt-relaxed-constexpr $flags -c $f.cu -o $out/obj/$f.o &
  done
  wait
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libgrnnd_b200.so $out/obj/*.o -lcudart
  rm -rf $out/obj
  echo built $out
done
