"""Small-M (decode-only batch) K3 GEMM vs cuBLAS, weights cold in L2 (flushed before every
timed launch) — the weight-streaming regime (dev tool). usage: gemm_small_m.py [M ...]"""
import os, sys, math, statistics
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
from paper_2403_02310_b200 import gpu

Ms = [int(x) for x in sys.argv[1:]] or [1, 32]
f = gpu.HybridForward(gpu.ModelShape("s", 1, 256, 4, 2, 64, 256, 512))
st = f.torch_stream()
flush = torch.empty(64 * 1024 * 1024, device="cuda", dtype=torch.float32)  # 256 MB > L2
shapes = [("qkv", 6144, 4096, 0), ("o", 4096, 4096, 1), ("gate_up", 28672, 4096, 2), ("down", 4096, 14336, 1)]


def timed(fn, reps=15):
    ts = []
    for _ in range(reps):
        with torch.cuda.stream(st):
            flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts) * 1e3


for M in Ms:
    for name, N, K, epi in shapes:
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        B = (torch.randn(N, K, device="cuda") / math.sqrt(K)).to(torch.bfloat16)
        D = torch.zeros(M, N // 2 if epi == 2 else N, device="cuda", dtype=torch.float32 if epi in (1, 3) else torch.bfloat16)
        wbytes = N * K * 2
        ours = timed(lambda: gpu.gpu_lib().ss_k_gemm(f.handle, A.data_ptr(), B.data_ptr(), D.data_ptr(), M, N, K, epi))
        with torch.cuda.stream(st):
            cub = timed(lambda: torch.matmul(A, B.T))
        print(f"M={M:3d} {name:8s} ours {ours:7.1f} us ({wbytes/ours/1e3:6.0f} GB/s)  cublas {cub:7.1f} us "
              f"({wbytes/cub/1e3:6.0f} GB/s)  splits={os.environ.get('SS_GEMM_SPLITS','auto')}", flush=True)
