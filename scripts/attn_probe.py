"""Attention kernel time per launch for batch compositions around the canonical batch (dev tool)."""
import os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_2403_02310_b200 import gpu, host

name = sys.argv[1] if len(sys.argv) > 1 else "mistral7b"
shape = gpu.MODELS[name].with_layers(2)
f = gpu.HybridForward(shape, weight_seed=1234)
f.kv_alloc(20000)
D, P = "decode", "prefill"
cases = {
    "canonical": [host.BatchEntry(i, D, 1, 4096) for i in range(32)] + [host.BatchEntry(32, P, 480, 0)],
    "decodes32": [host.BatchEntry(i, D, 1, 4096) for i in range(32)],
    "chunk480@0": [host.BatchEntry(0, P, 480, 0)],
    "chunk480@2048": [host.BatchEntry(0, P, 480, 2048)],
    "chunk2016@0": [host.BatchEntry(0, P, 2016, 0)],
    "decodes64": [host.BatchEntry(i, D, 1, 4096) for i in range(64)],
    "decodes37": [host.BatchEntry(i, D, 1, 4096) for i in range(37)],  # 296 pairs: 2 per SM
    "decodes19": [host.BatchEntry(i, D, 1, 4096) for i in range(19)],
    "decodes32@8k": [host.BatchEntry(i, D, 1, 8192) for i in range(32)],
}
only = os.environ.get("ONLY")
for cname, ents in cases.items():
    if only and cname not in only.split(","):
        continue
    d = host.Descriptor.build(ents, vocab=shape.vocab)
    f.fill_descriptor_prefixes(d, seed=5)
    b = f.upload(d)
    for _ in range(3):
        f.enqueue(b)
    f.synchronize()
    f.set_profiling(True)
    f.kernel_times(reset=True)
    for _ in range(5):
        f.enqueue(b)
    kt = f.kernel_times(reset=True)
    f.set_profiling(False)
    a = kt.get("attention", (0, 0))
    c = kt.get("attn_combine", (0, 0))
    kvb = sum((e.prefix_tokens + e.chunk_tokens) for e in ents) * shape.num_kv_heads * shape.head_dim * 4
    us = a[0] / max(a[1], 1) * 1e3
    print(f"{cname:14s} attention {us:7.1f} us/launch ({kvb/us/1e3:6.0f} GB/s K+V)  combine {c[0]/max(c[1],1)*1e3:6.1f} us", flush=True)
    b.free()
