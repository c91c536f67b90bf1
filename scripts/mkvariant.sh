#!/bin/bash
# Build the current tree's libss_gpu.so into build_variants/<name> (extra nvcc flags after the name).
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p build_variants/$name
nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
  --expt-relaxed-constexpr -Iinclude -Ipaper_2403_02310_b200/csrc/gpu "$@" -shared -cudart static \
  -o build_variants/$name/libss_gpu.so paper_2403_02310_b200/csrc/gpu/*.cu -ldl -lpthread -lrt 2>&1 | grep -E " error" ; true
