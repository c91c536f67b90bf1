"""Microbenchmark of the K3 GEMM on the Mistral tau=512 projection shapes (dev tool)."""
import os, sys, math
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
from paper_2403_02310_b200 import gpu

f = gpu.HybridForward(gpu.ModelShape("s", 1, 256, 4, 2, 64, 256, 512))
shapes = [("qkv", 512, 6144, 4096, 0), ("o", 512, 4096, 4096, 1), ("gate_up", 512, 28672, 4096, 2),
          ("down", 512, 4096, 14336, 1), ("lm_head", 33, 32000, 4096, 3), ("qkv2048", 2048, 6144, 4096, 0),
          ("gu2048", 2048, 28672, 4096, 2)]
st = f.torch_stream()
for name, M, N, K, epi in shapes:
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda") / math.sqrt(K)).to(torch.bfloat16)
    D = torch.zeros(M, N // 2 if epi == 2 else N, device="cuda", dtype=torch.float32 if epi in (1, 3) else torch.bfloat16)
    for _ in range(3):
        f.k_gemm(A, B, D, M, N, K, epi)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    e0.record(st)
    for _ in range(n):
        gpu.gpu_lib().ss_k_gemm(f.handle, A.data_ptr(), B.data_ptr(), D.data_ptr(), M, N, K, epi)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"{name:8s} M={M:5d} N={N:6d} K={K:6d} bn={os.environ.get('SS_GEMM_BN','auto'):4s} {ms*1e3:8.1f} us  {2*M*N*K/ms/1e9:7.1f} TFLOP/s", flush=True)
