#!/bin/bash
# Library variants x environment settings on ONE box (dev tool): for each round, each
# build_variants/<name>/libss_gpu.so runs scripts/ab_env.py with the given AB settings.
# usage: AB='SS_GEMM_DSM=1' TAU=32 NDEC=32 ab_lib_env.sh R name1 name2 ...
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
R="$1"; shift
cp paper_2403_02310_b200/libss_gpu.so /tmp/libss_gpu.orig.so
for r in $(seq 1 $R); do
  for v in "$@"; do
    cp build_variants/$v/libss_gpu.so paper_2403_02310_b200/libss_gpu.so
    timeout 600 python scripts/ab_env.py 2>&1 | grep median | sed "s/^/$v /"
  done
done
cp /tmp/libss_gpu.orig.so paper_2403_02310_b200/libss_gpu.so
