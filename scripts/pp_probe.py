"""Pipeline stages' device times on one B200 (dev probe): the canonical tau=512 batch through
PP = 1, 2, 4 stage contexts of the full Mistral-7B-shaped model; per-stage times (each from its
hand-off to its end), their sum against the unpipelined forward = the hand-off cost."""
import os
import statistics
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_2403_02310_b200 import gpu, host

shape = gpu.MODELS[os.environ.get("MODEL", "mistral7b")]
d = host.Descriptor.canonical(512, 32, 4096, 0, vocab=shape.vocab, token_seed=1)
f = gpu.HybridForward(shape, weight_seed=1234)
f.set_graphs(False)
f.kv_alloc(d.pool_blocks)
f.fill_descriptor_prefixes(d, seed=5)
ts = [f.forward(d, logits=False)[2] for _ in range(12)][2:]
print(f"# {shape.name} tau=512 canonical batch, ss_forward_hybrid / ss_forward_pipeline device ms (median of 10)")
print(f"  pp=1: {statistics.median(ts):.3f} ms (eager launches)")
f.close()
for pp in (2, 4):
    g = gpu.PipelineGroup(shape, pp, weight_seed=1234)
    g.kv_alloc(d.pool_blocks)
    g.fill_descriptor_prefixes(d, seed=5)
    rows = []
    for _ in range(12):
        g.forward(d, logits=False)
        rows.append(list(g.stage_ms))
    rows = rows[2:]
    med = [statistics.median(r[i] for r in rows) for i in range(pp)]
    print(f"  pp={pp}: stages " + ", ".join(f"{x:.3f}" for x in med) + f" ms; sum {sum(med):.3f}, max {max(med):.3f}")
    g.close()
