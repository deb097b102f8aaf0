#!/bin/bash
# build a development variant of libhc.so: tools/build_variant.sh <name> <extra nvcc flags...>
NAME=$1; shift
mkdir -p variants
/usr/local/cuda/bin/nvcc -shared -Xcompiler -fPIC -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a "$@" \
  -o variants/libhc_$NAME.so paper_1608_00206_b200/csrc/hc_api.cu
