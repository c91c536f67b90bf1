cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "gemm" 2>&1 | tail -3
SS_GEMM_SK=4 timeout 600 python -m pytest tests/test_gpu_forward.py -x -q 2>&1 | tail -3
CANDS="4,256;4,128;3,256;0,256;0,128" python scripts/gemm_class_sweep.py mistral7b 512 8 2>&1 | grep -E "^(default|0,|3,|4,)"
CANDS="4,256;4,128;3,256;0,256;0,128" python scripts/gemm_class_sweep.py llama70b:8 512 6 2>&1 | grep -E "^(default|0,|3,|4,)"
