#!/bin/bash
# Run probe_forward with each library variant under build_variants/<name>/libss_gpu.so (dev tool).
# usage: variants.sh "<probe args>" name1 name2 ...
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
args="$1"; shift
cp paper_2403_02310_b200/libss_gpu.so /tmp/libss_gpu.orig.so
for v in "$@"; do
  cp build_variants/$v/libss_gpu.so paper_2403_02310_b200/libss_gpu.so
  echo "== $v"
  timeout 300 python scripts/probe_forward.py $args 2>&1 | grep -E "ms/iter|gemm|attention|combine"
done
cp /tmp/libss_gpu.orig.so paper_2403_02310_b200/libss_gpu.so
