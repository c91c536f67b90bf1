"""GEMM main-loop scaling vs occupancy WITH the clock and power during each setting (dev probe):
each G (CTA pairs) runs the gate/up projection (M = 512, M-lockstep stream-K) back to back for
~1.5 s while nvidia-smi samples the SM clock and board power; per-k-block time per pair at
the measured clock separates the power-capped clock from the shared L2 -> SM bound."""
import math
import os
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch

from paper_2403_02310_b200 import gpu

M, N, K, epi = 512, 28672, 4096, 2
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
B = (torch.randn(N, K, device="cuda") / math.sqrt(K)).to(torch.bfloat16)
D = torch.zeros(M, N // 2, device="cuda", dtype=torch.bfloat16)
kbt = (M // 256) * (N // 256) * (K // 64)


def sample(stop, out):
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                           capture_output=True, text=True)
        try:
            c, p = r.stdout.strip().split(",")
            out.append((float(c), float(p)))
        except Exception:
            pass
        time.sleep(0.05)


print("# gate/up M=512 N=28672 K=4096, M-lockstep stream-K, back-to-back launches")
CASES = [(g, "0") for g in (74, 48, 24, 12)]
if os.environ.get("MC_CASES"):  # weight-tile multicast (4-CTA clusters) against unicast at equal pair counts
    CASES = [(74, "0"), (66, "0"), (66, "1"), (48, "0"), (48, "1")]
for G, mc in CASES:
    os.environ.update({"SS_GEMM_MAXG": str(G), "SS_GEMM_SK": "3", "SS_GEMM_BN": "256", "SS_GEMM_CG": "2",
                       "SS_GEMM_MC": mc})
    f = gpu.HybridForward(gpu.ModelShape("s", 1, 256, 4, 2, 64, 256, 512))
    st = torch.cuda.ExternalStream(f.stream_ptr)
    lib = gpu.gpu_lib()
    for _ in range(5):
        lib.ss_k_gemm(f._h, A.data_ptr(), B.data_ptr(), D.data_ptr(), M, N, K, epi)
    torch.cuda.synchronize()
    samples, stop = [], threading.Event()
    th = threading.Thread(target=sample, args=(stop, samples))
    th.start()
    n = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    e0.record(st)
    while time.time() - t0 < 1.5:
        for _ in range(50):
            lib.ss_k_gemm(f._h, A.data_ptr(), B.data_ptr(), D.data_ptr(), M, N, K, epi)
        n += 50
        torch.cuda.synchronize()
    e1.record(st)
    torch.cuda.synchronize()
    stop.set()
    th.join()
    us = e0.elapsed_time(e1) * 1e3 / n
    mhz = sorted(c for c, _ in samples)[len(samples) // 2] if samples else float("nan")
    w = sorted(p for _, p in samples)[len(samples) // 2] if samples else float("nan")
    per = us / (kbt / G)
    print(f"  G={G:3d} mc={mc}: {us:7.1f} us/launch, {per:.3f} us per k-block per pair at {mhz:.0f} MHz / {w:.0f} W "
          f"-> {per * mhz / 1965:.3f} us at 1965 MHz-equivalent cycles", flush=True)
    f.close()
