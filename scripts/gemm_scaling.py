"""Does the K3 main loop slow down as more CTA pairs run it? (dev probe: L2->SM / power bound)
For each G (CTA pairs allowed, SS_GEMM_MAXG), times one projection launch (events, L2 flushed)
with M-lockstep stream-K (balanced across any G) and reports the time per 64-wide k-block of
one 256 x 256 tile per pair: flat = per-SM bound, rising with G = shared-resource bound."""
import math
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch

from paper_2403_02310_b200 import gpu

shapes = [("gate_up", 512, 28672, 4096, 2), ("down", 512, 4096, 14336, 1), ("gate_up", 2048, 28672, 4096, 2)]
flush = torch.empty(512 * 1024 * 1024 // 4, device="cuda", dtype=torch.float32)
for name, M, N, K, epi in shapes:
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda") / math.sqrt(K)).to(torch.bfloat16)
    D = torch.zeros(M, N // 2 if epi == 2 else N, device="cuda",
                    dtype=torch.float32 if epi == 1 else torch.bfloat16)
    tiles = ((M + 255) // 256) * ((N + 255) // 256)
    kbt = tiles * (K // 64)
    for G in (74, 64, 48, 37, 24, 12):
        os.environ.update({"SS_GEMM_MAXG": str(G), "SS_GEMM_SK": "3", "SS_GEMM_BN": "256", "SS_GEMM_CG": "2"})
        f = gpu.HybridForward(gpu.ModelShape("s", 1, 256, 4, 2, 64, 256, 512))
        st = torch.cuda.ExternalStream(f.stream_ptr)
        ts = []
        for i in range(8):
            flush.fill_(float(i))
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            assert gpu.gpu_lib().ss_k_gemm(f._h, A.data_ptr(), B.data_ptr(), D.data_ptr(), M, N, K, epi) == 0
            e1.record(st)
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1) * 1e3)
        f.close()
        t = sorted(ts)[len(ts) // 2]
        print(f"{name:8s} M={M:5d} G={G:3d}: {t:8.1f} us  -> {t / (kbt / G):6.3f} us per k-block per pair, "
              f"{2 * M * N * K / t / 1e6:7.1f} TF/s", flush=True)
