#!/bin/bash
# GEMM schedule/tile sweep on the projection shapes (dev tool).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
SS_GEMM_DEBUG=1 timeout 120 python scripts/gemm_bench.py 2>&1 | grep -E "resident|TFLOP" | sort -u | head -40
for sk in 0 1; do for bn in 256 224 192 128; do
  echo "== SK=$sk BN=$bn"; SS_GEMM_SK=$sk SS_GEMM_BN=$bn SS_GEMM_CG=2 timeout 120 python scripts/gemm_bench.py 2>&1 | grep TFLOP
done; done
