"""A/B of dev tuning environment settings on the canonical batch (dev tool).
  AB='SS_ATTN_PF_PAGES=0;SS_ATTN_PF_PAGES=32 SS_GEMM_MC=1' TAU=512 python scripts/ab_env.py
Each setting gets its own context (the tuning is read at ss_create); settings are timed in
interleaved rounds (ROUNDS x STEPS back-to-back forwards, CUDA events, graphs on), median."""
import os
import statistics
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch

from paper_2403_02310_b200 import gpu, host

MODEL = os.environ.get("MODEL", "mistral7b")
shape = gpu.MODELS[MODEL]
if os.environ.get("LAYERS"):
    shape = shape.with_layers(int(os.environ["LAYERS"]))
TAU = int(os.environ.get("TAU", "512"))
PREFIX = int(os.environ.get("PREFIX", "0"))
NDEC = int(os.environ.get("NDEC", "32"))
ROUNDS, STEPS = int(os.environ.get("ROUNDS", "3")), int(os.environ.get("STEPS", "20"))
settings = [s for s in os.environ["AB"].split(";")]
if NDEC > 0 and TAU > NDEC:
    d = host.Descriptor.canonical(TAU, NDEC, 4096, PREFIX, vocab=shape.vocab, token_seed=1)
else:
    d = host.Descriptor.build([host.BatchEntry(i, "decode", 1, 4096) for i in range(NDEC)], vocab=shape.vocab, token_seed=1)
ctxs = []
for st in settings:
    kv = dict(x.split("=", 1) for x in st.split() if x)  # space-separated KEY=VALUE pairs
    old = {k: os.environ.get(k) for k in kv}
    os.environ.update(kv)
    f = gpu.HybridForward(shape, weight_seed=1234)
    for k, v in old.items():
        if v is None:
            os.environ.pop(k)
        else:
            os.environ[k] = v
    f.kv_alloc(d.pool_blocks)
    f.fill_descriptor_prefixes(d, seed=5)
    ctxs.append((st, f, f.upload(d)))
res = {st: [] for st in settings}
for r in range(ROUNDS):
    for st, f, b in ctxs:
        s = f.torch_stream()
        for _ in range(3):
            f.enqueue(b)
        f.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(STEPS):
            f.enqueue(b)
        e1.record(s)
        f.synchronize()
        res[st].append(e0.elapsed_time(e1) / STEPS)
print(f"# {MODEL} L={shape.num_layers} tau={TAU} ndec={NDEC} prefix={PREFIX}: ms/step per round")
for st in settings:
    print(f"  {st or '(default)':40s} median {statistics.median(res[st]):7.3f}  " + " ".join(f"{x:7.3f}" for x in res[st]))
