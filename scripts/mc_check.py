"""Weight-tile multicast (MC = 2) GEMMs vs torch (dev check): correctness and time, MC on/off."""
import math
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch

from paper_2403_02310_b200 import gpu

flush = torch.empty(512 * 1024 * 1024 // 4, device="cuda", dtype=torch.float32)
shapes = [("qkv", 512, 6144, 4096, 0), ("o", 512, 4096, 4096, 0), ("gate_up", 512, 28672, 4096, 2),
          ("down", 512, 4096, 14336, 0), ("down_resadd", 512, 4096, 14336, 1), ("gate_up", 2048, 28672, 4096, 2),
          ("qkv", 2048, 6144, 4096, 0), ("down", 2048, 4096, 14336, 0), ("o", 300, 4096, 4096, 0)]
ctxs = {}
for mc in ("1", "0"):  # SS_GEMM_MC=1 enables the multicast variant
    os.environ["SS_GEMM_MC"] = mc
    ctxs[mc] = gpu.HybridForward(gpu.ModelShape("s", 1, 256, 4, 2, 64, 256, 512))
for name, M, N, K, epi in shapes:
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda") / math.sqrt(K)).to(torch.bfloat16)
    ref = A.float() @ B.float().t()
    if epi == 2:
        g = ref.view(M, N // 64, 2, 32)
        ref = (torch.nn.functional.silu(g[:, :, 0]) * g[:, :, 1]).reshape(M, N // 2)
    res = {}
    for mc, f in ctxs.items():
        st = torch.cuda.ExternalStream(f.stream_ptr)
        ts = []
        for i in range(6):
            D = torch.zeros(M, N // 2 if epi == 2 else N, device="cuda", dtype=torch.float32 if epi == 1 else torch.bfloat16)
            flush.fill_(float(i))
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            assert gpu.gpu_lib().ss_k_gemm(f._h, A.data_ptr(), B.data_ptr(), D.data_ptr(), M, N, K, epi) == 0, \
                gpu.gpu_lib().ss_last_error(f._h)
            e1.record(st)
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1) * 1e3)
        err = float((D.float() - ref).norm() / ref.norm())
        res[mc] = (sorted(ts)[len(ts) // 2], err, D.clone())
    same = bool(torch.equal(res["1"][2], res["0"][2]))
    print(f"{name:12s} M={M:5d} N={N:6d} K={K:6d}: MC {res['1'][0]:7.1f} us (rel {res['1'][1]:.1e}) | "
          f"no-MC {res['0'][0]:7.1f} us (rel {res['0'][1]:.1e}) | bitwise equal {same}", flush=True)
