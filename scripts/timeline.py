"""Device timeline of one hybrid forward (dev tool): every kernel's start/end from CUPTI
(torch.profiler sees the library's kernels too), so PDL overlap between consecutive kernels
and the idle gaps between them are measured, not inferred from per-launch events.

  MODEL=mistral7b LAYERS=4 python scripts/timeline.py > profiles/r02/timeline_mistral7b.txt

Prints, per kernel of one steady-state layer: start and end relative to the layer's first
kernel, duration, and the overlap with (negative) or gap after (positive) the previous kernel's
end; then per-class sums over all layers and the step's busy / idle time.
"""
import collections
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2403_02310_b200 import gpu, host

MODEL = os.environ.get("MODEL", "mistral7b")
shape = gpu.MODELS[MODEL]
if os.environ.get("LAYERS"):
    shape = shape.with_layers(int(os.environ["LAYERS"]))
TAU = int(os.environ.get("TAU", "512"))
PREFIX = int(os.environ.get("PREFIX", "0"))
GRAPHS = os.environ.get("GRAPHS", "1") == "1"

f = gpu.HybridForward(shape, weight_seed=1234)
NDEC = int(os.environ.get("NDEC", "32"))
if os.environ.get("DECODE_ONLY"):  # NDEC decodes at 4096, no chunk (the TBT-critical step)
    d = host.Descriptor.build([host.BatchEntry(i, "decode", 1, 4096) for i in range(NDEC)], vocab=shape.vocab,
                              token_seed=1)
else:
    d = host.Descriptor.canonical(TAU, NDEC, 4096, PREFIX, vocab=shape.vocab, token_seed=1)
f.kv_alloc(d.pool_blocks)
f.fill_descriptor_prefixes(d, seed=5)
b = f.upload(d)
f.set_graphs(GRAPHS)
for _ in range(5):
    f.enqueue(b)
f.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        f.enqueue(b)
    f.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and e.device_time_total > 0]
# kernels of the last forward
ker = sorted([(e.time_range.start, e.time_range.end, e.name) for e in ev if "Memcpy" not in e.name
              and "Memset" not in e.name])
per = len(ker) // 3
ker = ker[-per:]


def cls(n):
    for key, c in (("embed", "embed"), ("argmax", "argmax"), ("rmsnorm", "rmsnorm"), ("combine", "attn_combine"),
                   ("attention_kernel", "attention"), ("gemm", "gemm")):
        if key in n:
            return c
    return n[:40]


names = []
for s, e, n in ker:
    c = cls(n)
    if c == "gemm":
        epi = n.split("gemm_tcgen05_kernel<")[1].split(",")[2].strip() if "gemm_tcgen05_kernel<" in n else "?"
        c = {"4": "gemm_qkv", "1": "gemm_resadd(o|down)", "2": "gemm_gate_up", "3": "lm_head", "0": "gemm_bf16"}.get(epi, "gemm")
    if c == "attention":
        c = "attention(tc)" if ", 0>" not in n and "0>" not in n.split(",")[-1] else "attention(decode)"
    names.append(c)
t0 = ker[0][0]
span = ker[-1][1] - t0
busy = 0.0
cur_s, cur_e = None, None
for s, e, _ in ker:
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
busy += cur_e - cur_s
print(f"# {MODEL} L={shape.num_layers} tau={TAU} chunk prefix {PREFIX}, graphs {'on' if GRAPHS else 'off'}: "
      f"{len(ker)} kernels, step span {span:.1f} us, device busy {busy:.1f} us, idle {span - busy:.1f} us")
# one steady-state layer: the kernels between the 2nd and 3rd QKV GEMM
qidx = [i for i, c in enumerate(names) if c == "gemm_qkv"]
if len(qidx) >= 3:
    a, z = qidx[1], qidx[2]
    base = ker[a][0]
    print(f"# layer 1 (kernels {a}..{z - 1}): start / end relative to the layer's QKV start, us")
    prev_end = ker[a - 1][1]
    for i in range(a, z):
        s, e, n = ker[i]
        print(f"  {names[i]:22s} start {s - base:8.1f} end {e - base:8.1f} dur {e - s:7.1f}  "
              f"{'gap' if s >= prev_end else 'overlap'} {abs(s - prev_end):6.1f}")
        prev_end = max(prev_end, e)
    print(f"  layer span {ker[z][0] - base:.1f} us")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for (s, e, _), c in zip(ker, names):
    tot[c] += e - s
    cnt[c] += 1
print("# per class over the step: kernel-duration sum (us), launches")
for c in sorted(tot, key=lambda k: -tot[k]):
    print(f"  {c:22s} {tot[c]:9.1f} {cnt[c]:5d}")
