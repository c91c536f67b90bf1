"""Does splitting the hybrid batch into a decode stream and a chunk stream pay on B200? (dev tool)

Measures, Mistral-7B-shaped at full depth, the canonical tau = 512 batch (32 decodes @ 4096 +
a 480-token chunk @ 0):
  unified     the one hybrid forward (decode rows ride in the chunk's projection GEMMs)
  decode      the 32 decodes alone (the M = 32 projections stream every weight again)
  chunk       the 480-token chunk alone
  concurrent  decode and chunk forwards in two contexts on two streams at once (the
              hardware scheduler shares the SMs; nano-batch overlap of HBM-bound decode
              attention with tensor-bound chunk GEMMs, paying one extra weight read)
CUDA events, device time, median of REPS.
"""
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch

from paper_2403_02310_b200 import gpu, host

REPS = int(os.environ.get("REPS", "20"))
shape = gpu.MODELS[os.environ.get("MODEL", "mistral7b")]
if os.environ.get("LAYERS"):
    shape = shape.with_layers(int(os.environ["LAYERS"]))

uni = host.Descriptor.canonical(512, 32, 4096, 0, vocab=shape.vocab, token_seed=1)
dec = host.Descriptor.build([host.BatchEntry(i, "decode", 1, 4096) for i in range(32)], vocab=shape.vocab, token_seed=1)
chk = host.Descriptor.build([host.BatchEntry(100, "prefill", 480, 0)], completes=[True], vocab=shape.vocab, token_seed=1)


def ctx_for(d):
    f = gpu.HybridForward(shape, weight_seed=1234)
    f.kv_alloc(d.pool_blocks)
    f.fill_descriptor_prefixes(d, seed=5)
    return f, f.upload(d)


def time_one(f, b):
    s = torch.cuda.ExternalStream(f.stream_ptr)
    ts = []
    for i in range(REPS + 3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        f.enqueue(b)
        e1.record(s)
        s.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def time_pair(fa, ba, fb, bb):
    sa = torch.cuda.ExternalStream(fa.stream_ptr)
    sb = torch.cuda.ExternalStream(fb.stream_ptr)
    ts = []
    for i in range(REPS + 3):
        torch.cuda.synchronize()
        e0, ea, eb = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(sa)
        sb.wait_event(e0)
        fa.enqueue(ba)
        fb.enqueue(bb)
        ea.record(sa)
        eb.record(sb)
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(max(e0.elapsed_time(ea), e0.elapsed_time(eb)))
    ts.sort()
    return ts[len(ts) // 2]


res = {}
f, b = ctx_for(uni)
f.set_graphs(False)
res["unified"] = time_one(f, b)
del b
f.close()
fd, bd = ctx_for(dec)
fc, bc = ctx_for(chk)
fd.set_graphs(False)
fc.set_graphs(False)
res["decode"] = time_one(fd, bd)
res["chunk"] = time_one(fc, bc)
res["concurrent"] = time_pair(fd, bd, fc, bc)
print(f"# {shape.name} L={shape.num_layers}, device ms per step (median of {REPS})")
for k, v in res.items():
    print(f"  {k:11s} {v:8.3f} ms")
print(f"  sum(decode, chunk) {res['decode'] + res['chunk']:8.3f} ms")
