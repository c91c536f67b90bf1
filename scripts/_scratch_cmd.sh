cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_forward.py tests/test_gpu_tp_local.py tests/test_gpu_chain.py -q -x -p no:cacheprovider > gpurun_out/test_qkv.txt 2>&1
tail -4 gpurun_out/test_qkv.txt
AB=';SS_GEMM_QKV=0,256;SS_GEMM_QKV=2,192,2' ROUNDS=3 timeout 600 python scripts/ab_env.py > gpurun_out/ab_qkv.txt 2>&1
tail -4 gpurun_out/ab_qkv.txt
SS_GEMM_DEBUG=1 LAYERS=2 timeout 120 python scripts/chain_check.py 2>&1 | grep "epi=4" | sort | uniq | head
