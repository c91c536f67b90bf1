"""Which kernels cuBLAS (torch.matmul) runs for the projection shapes (dev tool): names encode the
tile / cluster choices (nvjet_*), durations from CUPTI."""
import torch
from torch.profiler import ProfilerActivity, profile

for M in (32, 512, 2048):
    for name, N, K in (("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336)):
        A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
        B = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
        C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        for _ in range(3):
            torch.matmul(A, B.t(), out=C)
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            torch.matmul(A, B.t(), out=C)
            torch.cuda.synchronize()
        ks = [(e.name, e.time_range.end - e.time_range.start) for e in prof.events()
              if e.device_type == torch.autograd.DeviceType.CUDA]
        print(f"{name:8s} M={M:5d}: " + "; ".join(f"{n} {d:.1f}us" for n, d in ks), flush=True)
