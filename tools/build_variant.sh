#!/bin/bash
# build an experimental variant of libpolylla.so with extra -D flags: tools/build_variant.sh NAME -DFLAG ...
name=$1; shift
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false "$@" \
  -Xcompiler -fPIC,-fvisibility=hidden -shared -I include -o paper_2403_14723_b200/libpolylla_$name.so \
  paper_2403_14723_b200/csrc/*.cu
