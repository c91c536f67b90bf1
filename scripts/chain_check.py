"""Fused projection chain vs separate launches (dev check): logits agreement and step time.
  MODEL=mistral7b LAYERS=2 python scripts/chain_check.py"""
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import numpy as np
import torch

from paper_2403_02310_b200 import gpu, host

MODEL = os.environ.get("MODEL", "mistral7b")
shape = gpu.MODELS[MODEL]
if os.environ.get("LAYERS"):
    shape = shape.with_layers(int(os.environ["LAYERS"]))
TAU = int(os.environ.get("TAU", "512"))
PREFIX = int(os.environ.get("PREFIX", "0"))
REPS = int(os.environ.get("REPS", "20"))


DECODE = int(os.environ.get("DECODE", "0"))  # > 0: a decode-only batch of DECODE sequences @ 4096


def run(chain):
    os.environ["SS_CHAIN"] = ("2" if DECODE else "1") if chain else "0"
    f = gpu.HybridForward(shape, weight_seed=1234)
    if DECODE:
        d = host.Descriptor.build([host.BatchEntry(i, "decode", 1, 4096) for i in range(DECODE)], vocab=shape.vocab,
                                  token_seed=1)
    else:
        d = host.Descriptor.canonical(TAU, 32, 4096, PREFIX, vocab=shape.vocab, token_seed=1)
    f.kv_alloc(d.pool_blocks)
    f.fill_descriptor_prefixes(d, seed=5)
    lg, nt, _ = f.forward(d)
    lg2, _, _ = f.forward(d)
    b = f.upload(d)
    st = f.torch_stream()
    for _ in range(3):
        f.enqueue(b)
    f.synchronize()
    ts = []
    for _ in range(REPS):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        f.enqueue(b)
        e1.record(st)
        f.synchronize()
        ts.append(e0.elapsed_time(e1))
    b.free()
    f.close()
    return lg, lg2, sorted(ts)[len(ts) // 2]


a, a2, ta = run(False)
c, c2, tc = run(True)
rel = float(np.linalg.norm(c - a) / np.linalg.norm(a))
print(f"{MODEL} L={shape.num_layers} tau={TAU} prefix={PREFIX} decode-only={DECODE}: separate {ta:.3f} ms, chain {tc:.3f} ms; "
      f"rel-L2(chain vs separate) {rel:.2e}, top-1 agree {float((c.argmax(1) == a.argmax(1)).mean()):.3f}, "
      f"chain repeatable {bool((c == c2).all())}, separate repeatable {bool((a == a2).all())}")
