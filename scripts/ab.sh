#!/bin/bash
# A/B the forward time of library variants on ONE box (variance across boxes is
# several %): alternates build_variants/<name>/libss_gpu.so, R rounds (dev tool).
# usage: ab.sh "<probe_forward args>" R name1 name2 ...
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
args="$1"; R="$2"; shift 2
cp paper_2403_02310_b200/libss_gpu.so /tmp/libss_gpu.orig.so
for r in $(seq 1 $R); do
  for v in "$@"; do
    cp build_variants/$v/libss_gpu.so paper_2403_02310_b200/libss_gpu.so
    echo "$v $(timeout 300 python scripts/probe_forward.py $args 2>&1 | grep -E 'tau=' | sed 's/.*L=[0-9]*: //')"
  done
done
cp /tmp/libss_gpu.orig.so paper_2403_02310_b200/libss_gpu.so
