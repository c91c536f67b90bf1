echo "== default"; python scripts/gemm_bench.py 2>&1 | head -4
echo "== bn256 sk1"; SS_GEMM_BN=256 SS_GEMM_SK=1 python scripts/gemm_bench.py 2>&1 | head -4
echo "== bn256 sk0"; SS_GEMM_BN=256 SS_GEMM_SK=0 python scripts/gemm_bench.py 2>&1 | head -4
echo "== bn256 split2"; SS_GEMM_BN=256 SS_GEMM_SPLITS=2 python scripts/gemm_bench.py 2>&1 | head -4
echo "== bn224 sk1"; SS_GEMM_BN=224 SS_GEMM_SK=1 python scripts/gemm_bench.py 2>&1 | head -4
echo "== bn128 sk1"; SS_GEMM_BN=128 SS_GEMM_SK=1 python scripts/gemm_bench.py 2>&1 | head -4
