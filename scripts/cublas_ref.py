"""cuBLAS (torch.matmul) times on the same projection shapes, as a practical ceiling reference (dev tool)."""
import torch
shapes = [("qkv", 512, 6144, 4096), ("o", 512, 4096, 4096), ("gate_up", 512, 28672, 4096), ("down", 512, 4096, 14336),
          ("gu2048", 2048, 28672, 4096)]
for name, M, N, K in shapes:
    A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
    for _ in range(5):
        C = A @ B.T
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        C = A @ B.T
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"cublas {name:8s} M={M} N={N} K={K}: {ms*1e3:7.1f} us {2*M*N*K/ms/1e9:7.1f} TFLOP/s", flush=True)
