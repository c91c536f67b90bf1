"""K3 projection GEMMs against cuBLAS (torch.matmul) on the same shapes, same conditions (dev tool).

Both arms: bf16 A[M,K] . B[N,K]^T, fresh inputs resident in HBM, L2 flushed (a 512 MB write)
before every timed launch, CUDA events around each launch on the launching stream, median of
REPS. Ours runs with the plain bf16-store epilogue (EPI_BF16; SwiGLU for gate/up, whose output
is half as wide) through ss_k_gemm. Shapes: the Mistral-7B projections at the canonical
tau = 512 batch (M = 512), decode-only steps (M = 32) and tau = 2048 (M = 2048).
  python scripts/gemm_vs_cublas.py > profiles/r02/gemm_vs_cublas.txt
"""
import math
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch

from paper_2403_02310_b200 import gpu

REPS = int(os.environ.get("REPS", "30"))
PROJ = [("qkv", 6144, 4096, 0), ("o", 4096, 4096, 0), ("gate_up", 28672, 4096, 2), ("down", 4096, 14336, 0)]
MS = [int(m) for m in os.environ.get("MS", "32,512,2048").split(",")]

f = gpu.HybridForward(gpu.ModelShape("s", 1, 256, 4, 2, 64, 256, 512))
flush = torch.empty(512 * 1024 * 1024 // 4, device="cuda", dtype=torch.float32)
st = torch.cuda.Stream()
ours_stream = torch.cuda.ExternalStream(f.stream_ptr)


def timed(fn, stream):
    ts = []
    for i in range(REPS + 3):
        with torch.cuda.stream(stream):
            flush.fill_(float(i))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
        stream.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


print(f"# {torch.cuda.get_device_name()}  L2 flushed before every launch, median of {REPS}")
print(f"# {'shape':<10s} {'M':>5s} {'N':>6s} {'K':>6s} | {'ours us':>8s} {'TF/s':>7s} {'GB/s':>7s} | "
      f"{'cuBLAS us':>9s} {'TF/s':>7s} | ours/cuBLAS speed")
for M in MS:
    for name, N, K, epi in PROJ:
        A = (torch.randn(M, K, device="cuda")).to(torch.bfloat16)
        B = (torch.randn(N, K, device="cuda") / math.sqrt(K)).to(torch.bfloat16)
        D = torch.empty(M, N // 2 if epi == 2 else N, device="cuda", dtype=torch.bfloat16)
        C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        torch.cuda.synchronize()

        def ours():  # straight through the C ABI on the library stream (no host fence inside the timing)
            assert gpu.gpu_lib().ss_k_gemm(f._h, A.data_ptr(), B.data_ptr(), D.data_ptr(), M, N, K, epi) == 0

        def cub():
            torch.matmul(A, B.t(), out=C)

        t_o = timed(ours, ours_stream)
        t_c = timed(cub, st)
        fl = 2.0 * M * N * K
        by = 2.0 * (M * K + N * K + M * (N // 2 if epi == 2 else N))
        print(f"  {name:<10s} {M:5d} {N:6d} {K:6d} | {t_o:8.1f} {fl / t_o / 1e6:7.1f} {by / t_o / 1e3:7.0f} | "
              f"{t_c:9.1f} {fl / t_c / 1e6:7.1f} | {t_c / t_o:5.2f}", flush=True)
