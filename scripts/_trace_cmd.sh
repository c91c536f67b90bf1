timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -2
cp build_variants/tnew/libss_gpu.so paper_2403_02310_b200/libss_gpu.so
echo "=== tnew"; python scripts/gemm_trace.py 2>&1 | grep -E "M=|seg 0|exit"
echo "=== tnew M32"; M=32 ONLY=qkv,o python scripts/gemm_trace.py 2>&1 | grep -E "M=|seg 0|exit"
bash scripts/ab.sh "mistral7b 512" 3 base new
