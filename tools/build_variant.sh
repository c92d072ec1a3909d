#!/bin/bash
# Build a tuning variant of the library: tools/build_variant.sh NAME -DMACRO=V ...
# -> paper_2303_14335_b200/lib/variants/libmpld_NAME.so (load with MPLD_LIB=...)
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p paper_2303_14335_b200/lib/variants
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC,-O2 -shared \
  -Iinclude "$@" -o paper_2303_14335_b200/lib/variants/libmpld_$name.so \
  paper_2303_14335_b200/csrc/kernels_graph.cu paper_2303_14335_b200/csrc/kernel_search.cu paper_2303_14335_b200/csrc/kernel_tile.cu paper_2303_14335_b200/csrc/mpld_api.cu
echo built $name
