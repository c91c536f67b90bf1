cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
AB=';SS_GEMM_O=2,128,3 SS_GEMM_DOWN=2,128,3 SS_GEMM_GATEUP=0,256;SS_GEMM_O=2,64,2 SS_GEMM_DOWN=2,64,2;SS_GEMM_GATEUP=3,64 SS_GEMM_DOWN=0,64' TAU=32 NDEC=32 ROUNDS=3 timeout 600 python scripts/ab_env.py > gpurun_out/ab_dec64.txt 2>&1
tail -6 gpurun_out/ab_dec64.txt
SS_GEMM_DEBUG=1 timeout 120 python -c "
import sys; sys.path.insert(0,'.')
from paper_2403_02310_b200 import gpu, host
s=gpu.MODELS['mistral7b'].with_layers(1)
d=host.Descriptor.build([host.BatchEntry(i,'decode',1,4096) for i in range(32)], vocab=s.vocab)
f=gpu.HybridForward(s); f.kv_alloc(d.pool_blocks); f.fill_descriptor_prefixes(d,seed=5); f.set_graphs(False); f.forward(d)
" 2>&1 | grep "gemm cg" | head -6
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k gemm > gpurun_out/test_gemm.txt 2>&1
tail -5 gpurun_out/test_gemm.txt
