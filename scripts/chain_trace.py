"""Per-item timeline of the fused projection chain inside the forward (dev tool).
  SS_CHAIN_TRACE=1 MODEL=mistral7b TAU=512 LAYER=1 python scripts/chain_trace.py
Columns per item (leader CTA, globaltimer ns): producer start / producer done / MMA start /
MMA done / epilogue start / tile published. Prints, per phase, its window and the medians of
producer issue time, MMA time, MMA start lag behind the producer and epilogue latency."""
import ctypes as C
import os
import sys

os.environ.setdefault("SS_CHAIN_TRACE", "1")
os.environ.setdefault("SS_CHAIN", "2" if int(os.environ.get("DECODE", "0")) else "1")
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import numpy as np

from paper_2403_02310_b200 import gpu, host

MODEL = os.environ.get("MODEL", "mistral7b")
shape = gpu.MODELS[MODEL]
if os.environ.get("LAYERS"):
    shape = shape.with_layers(int(os.environ["LAYERS"]))
TAU = int(os.environ.get("TAU", "512"))
LAYER = int(os.environ.get("LAYER", "1"))
lib = gpu.gpu_lib()
lib.ss_debug_chain_trace.restype = C.c_int
lib.ss_debug_chain_trace.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]

f = gpu.HybridForward(shape, weight_seed=1234)
f.set_graphs(False)
DECODE = int(os.environ.get("DECODE", "0"))  # > 0: decode-only batch (the single-CTA weight-streaming chain)
if DECODE:
    d = host.Descriptor.build([host.BatchEntry(i, "decode", 1, 4096) for i in range(DECODE)], vocab=shape.vocab,
                              token_seed=1)
    TAU = DECODE
else:
    d = host.Descriptor.canonical(TAU, 32, 4096, 0, vocab=shape.vocab, token_seed=1)
f.kv_alloc(d.pool_blocks)
f.fill_descriptor_prefixes(d, seed=5)
b = f.upload(d)
for _ in range(3):
    f.enqueue(b)
f.synchronize()
assert lib.ss_debug_chain_trace(f._h, None, -1) == 0
f.enqueue(b)
f.synchronize()
n = shape.num_layers * 4096 * 16
buf = np.zeros(n, np.uint64)
assert lib.ss_debug_chain_trace(f._h, buf.ctypes.data, n) == 0, gpu.gpu_lib().ss_last_error(f._h)
tr = buf.reshape(shape.num_layers, 4096, 16)[LAYER].astype(np.int64)
live = tr[:, 0] > 0
items = np.nonzero(live)[0]
t0 = tr[live][:, 0].min()
rel = lambda v: (v - t0) / 1e3
# phase boundaries from the chain's own item counts
h, ffn, T = shape.hidden, shape.ffn, TAU
nq, nkv, hd = shape.num_q_heads, shape.num_kv_heads, shape.head_dim
cg = 2 if T > 128 else 1
num_mt = (T + 128 * cg - 1) // (128 * cg)
S = [int(x) for x in os.environ.get("SS_CHAIN_S", "0,0,0,0").split(",")]
K = [nq * hd, h, ffn, h]
N = [h, 2 * ffn, h, (nq + 2 * nkv) * hd]
names = ["o", "gate_up", "down", "qkv"]
start = 0
print(f"# {MODEL} tau={TAU} layer {LAYER}: {len(items)} items, span {rel(tr[live][:, 5].max()):.1f} us "
      f"(from the first producer start)")
for p in range(4):
    nkb = (K[p] + 63) // 64
    tiles = num_mt * ((N[p] + 255) // 256)
    auto = max(1, (nkb + 32) // 64) if cg == 2 else max(1, min(nkb // 8, (148 + tiles - 1) // tiles))
    s = S[p] if S[p] > 0 else auto
    cnt = num_mt * ((N[p] + 255) // 256) * s
    sel = [i for i in items if start <= i < start + cnt]
    start += cnt
    if not sel:
        continue
    r = tr[sel]
    pub = r[r[:, 5] > 0]
    print(f"  {names[p]:8s} items {len(sel):4d} (splits {s}): producer start {rel(r[:, 0].min()):7.1f}..{rel(r[:, 0].max()):7.1f}"
          f"  MMA {rel(r[:, 2].min()):7.1f}..{rel(r[:, 3].max()):7.1f}  published {rel(pub[:, 5].min()) if len(pub) else -1:7.1f}..{rel(pub[:, 5].max()) if len(pub) else -1:7.1f}")
    print(f"           medians: producer issue {np.median(r[:, 1] - r[:, 0]) / 1e3:6.2f} us, MMA {np.median(r[:, 3] - r[:, 2]) / 1e3:6.2f} us, "
          f"MMA start - producer start {np.median(r[:, 2] - r[:, 0]) / 1e3:6.2f} us, epilogue start - MMA done {np.median(r[:, 4] - r[:, 3]) / 1e3:6.2f} us"
          + (f", published - epilogue start {np.median(pub[:, 5] - pub[:, 4]) / 1e3:6.2f} us" if len(pub) else ""))
if os.environ.get("DUMP"):
    for i in items:
        print(i, " ".join(f"{rel(v):7.1f}" if v > 0 else "     - " for v in tr[i, :16]))
