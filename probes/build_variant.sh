#!/bin/bash
# Build a libqpk.so variant with extra -D flags for A/B runs (probes/ab_engine.py):
#   probes/build_variant.sh probes/libs/lib_x.so -DQPK_TILE_GATHER_WARPS=4
out=$1; shift
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 \
  -shared -cudart static -I include "$@" -o "$out" paper_2308_00637_b200/csrc/qpk.cu 2>&1 | grep -i error
exit 0
