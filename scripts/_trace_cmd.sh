timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_forward.py -x -q 2>&1 | tail -2
for i in 1 2; do python scripts/probe_forward.py mistral7b 512 2>&1 | grep -E "ms/iter|gemm_qkv"; done
