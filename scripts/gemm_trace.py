"""Per-CTA timeline of one K3 GEMM launch (dev tool; needs the -DSS_GEMM_TRACE build).
usage: gemm_trace.py [cold | fwd]. Slots: 0 entry, 1 after pdl_wait, 2 first stage full, 3..6 end of
the MMA issue of segments 0..3, 7 exit (globaltimer ns). `fwd` traces each projection inside a
1-layer Mistral forward of the canonical batch (SLOW=n prints the n slowest CTAs)."""
import os, sys, math, ctypes as C
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import numpy as np
import torch
from paper_2403_02310_b200 import gpu

lib = gpu.gpu_lib()


def clear(epi=None):
    assert lib.ss_debug_gemm_trace(None, -1) == 0
    assert lib.ss_debug_gemm_trace(None, -2 if epi is None else -3 - epi) == 0


def report(name):
    tr = np.zeros((1024, 8), np.uint64)
    assert lib.ss_debug_gemm_trace(tr.ctypes.data_as(C.POINTER(C.c_ulonglong)), 1024) == 0
    tr = tr.astype(np.int64)
    t0 = tr[tr[:, 0] > 0, 0].min()
    live = tr[:, 0] >= t0  # this launch (older launches have earlier stamps)
    rows = tr[live]
    lead = rows[rows[:, 2] >= t0]
    rel = lambda v: (v - t0) / 1e3
    print(f"{name}: {len(rows)} CTAs, span {rel(rows[:, 7].max()):.1f} us")
    print(f"   pdl wait done med {np.median(rel(rows[:, 1])):6.1f} max {rel(rows[:, 1].max()):6.1f}")
    print(f"   first data   med {np.median(rel(lead[:, 2])):6.1f}")
    for j in range(4):
        v = lead[:, 3 + j]
        v = v[v >= t0]
        if len(v):
            print(f"   seg {j} MMA end: n={len(v):3d} min {rel(v.min()):6.1f} med {np.median(rel(v)):6.1f} max {rel(v.max()):6.1f}")
    t2 = np.zeros((1024, 16), np.uint64)
    assert lib.ss_debug_gemm_trace(t2.ctypes.data_as(C.POINTER(C.c_ulonglong)), 4096) == 0
    t2 = t2.astype(np.int64)[live]
    for j, nm in enumerate(["tfull seen (last seg)", "flags done (heads)", "epilogue done", "published (pieces)",
                              "staged 1st piece in", "staged done", "staged bar passed", "7", "8", "9", "10", "11",
                              "12", "13"]):
        v = t2[:, j]
        v = v[v >= t0]
        if len(v):
            print(f"   {nm:22s} n={len(v):3d} min {rel(v.min()):6.1f} med {np.median(rel(v)):6.1f} max {rel(v.max()):6.1f}")
    print(f"   exit         min {rel(rows[:, 7].min()):6.1f} med {np.median(rel(rows[:, 7])):6.1f} max {rel(rows[:, 7].max()):6.1f}")
    if os.environ.get("SLOW"):
        idx = np.nonzero(live)[0]
        order = idx[np.argsort(-tr[idx, 7])][: int(os.environ["SLOW"])]
        for b in order:
            st = ["%6.1f" % rel(v) if v >= t0 else "   -  " for v in tr[b]]
            s2 = ["%6.1f" % rel(v) if v >= t0 else "   -  " for v in t2[np.searchsorted(idx, b)]]
            print(f"   cta {b:3d}: " + " ".join(st) + " | " + " ".join(s2))


mode = sys.argv[1] if len(sys.argv) > 1 else ""
only = os.environ.get("ONLY")
if mode == "fwd":
    from paper_2403_02310_b200 import host
    shape = gpu.MODELS[os.environ.get("MODEL", "mistral7b")].with_layers(1)
    f = gpu.HybridForward(shape, weight_seed=1234)
    if os.environ.get("DECODE"):  # 32 decodes at 4096, no chunk (the TBT-critical step)
        d = host.Descriptor.build([host.BatchEntry(i, "decode", 1, 4096) for i in range(32)], vocab=shape.vocab)
    else:
        d = host.Descriptor.canonical(512, 32, 4096, 0, vocab=shape.vocab)
    f.kv_alloc(d.pool_blocks)
    f.fill_descriptor_prefixes(d, seed=5)
    b = f.upload(d)
    for name, epi in [("qkv", 4), ("gate_up", 2), ("o+down", 1)]:
        if only and name not in only.split(","):
            continue
        for _ in range(3):
            f.enqueue(b)
        f.synchronize()
        clear(epi)
        f.enqueue(b)
        f.synchronize()
        report(f"fwd {name} (last launch with epilogue {epi})")
    clear(None)
    sys.exit(0)

f = gpu.HybridForward(gpu.ModelShape("s", 1, 256, 4, 2, 64, 256, 512))
flush = torch.empty(512 * 1024 * 1024 // 4, device="cuda", dtype=torch.float32)
shapes = [("qkv", 512, 6144, 4096, 0), ("o", 512, 4096, 4096, 1), ("gate_up", 512, 28672, 4096, 2),
          ("down", 512, 4096, 14336, 1)]
if os.environ.get("M"):
    shapes = [(n, int(os.environ["M"]), N, K, e) for n, _, N, K, e in shapes]
for name, M, N, K, epi in shapes:
    if only and name not in only.split(","):
        continue
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda") / math.sqrt(K)).to(torch.bfloat16)
    pad = int(os.environ.get("SS_GEMM_LDO_PAD", "0"))
    D = torch.zeros(M, (N // 2 if epi == 2 else N) + pad, device="cuda", dtype=torch.float32 if epi in (1, 3) else torch.bfloat16)
    for _ in range(3):
        f.k_gemm(A, B, D, M, N, K, epi)
    if mode == "cold":
        flush.fill_(1.0)
    torch.cuda.synchronize()
    clear()
    f.k_gemm(A, B, D, M, N, K, epi)
    report(f"{name:8s} M={M} N={N} K={K}")
