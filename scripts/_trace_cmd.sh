timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -2
echo "== default"; python scripts/gemm_bench.py 2>&1 | head -4
echo "== bn256 split2"; SS_GEMM_BN=256 SS_GEMM_SPLITS=2 python scripts/gemm_bench.py 2>&1 | head -4
echo "== split4"; SS_GEMM_SPLITS=4 python scripts/gemm_bench.py 2>&1 | head -4
python scripts/probe_forward.py mistral7b 512 2>&1 | grep -E "ms/iter|gemm"
