"""Run one GEMM shape a few times (for ncu captures). usage: gemm_one.py M N K epi"""
import os, sys, math
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
from paper_2403_02310_b200 import gpu
M, N, K, epi = map(int, sys.argv[1:5])
f = gpu.HybridForward(gpu.ModelShape("s", 1, 256, 4, 2, 64, 256, 512))
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
B = (torch.randn(N, K, device="cuda") / math.sqrt(K)).to(torch.bfloat16)
D = torch.zeros(M, N // 2 if epi == 2 else N, device="cuda", dtype=torch.float32 if epi in (1, 3) else torch.bfloat16)
for _ in range(3):
    f.k_gemm(A, B, D, M, N, K, epi)
torch.cuda.synchronize()
