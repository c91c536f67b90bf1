"""Quick device-time probe of the canonical hybrid batch (dev tool)."""
import sys, time, os
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import numpy as np
import torch
from paper_2403_02310_b200 import gpu, host

name = sys.argv[1] if len(sys.argv) > 1 else "mistral7b"
tau = int(sys.argv[2]) if len(sys.argv) > 2 else 512
layers = int(sys.argv[3]) if len(sys.argv) > 3 else 0
shape = gpu.MODELS[name]
if layers:
    shape = shape.with_layers(layers)
t0 = time.time()
f = gpu.HybridForward(shape, weight_seed=1234)
print(f"create {time.time()-t0:.2f}s", flush=True)
d = host.Descriptor.canonical(tau, 32, 4096, 0, vocab=shape.vocab)
f.kv_alloc(d.pool_blocks)
t0 = time.time(); f.fill_descriptor_prefixes(d, seed=5); print(f"kv fill {time.time()-t0:.2f}s", flush=True)
lg, nt, ms = f.forward(d)
print("first forward ms", ms, "finite", np.isfinite(lg).all(), "tokens", nt[:8], flush=True)
b = f.upload(d)
st = f.torch_stream()
for _ in range(3):
    f.enqueue(b)
f.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
K = 10
e0.record(st)
for _ in range(K):
    f.enqueue(b)
e1.record(st)
f.synchronize()
tms = e0.elapsed_time(e1) / K
print(f"{name} tau={tau} L={shape.num_layers}: {tms:.3f} ms/iter, {tau/tms*1e3:.0f} tok/s", flush=True)
f.set_profiling(True)
f.kernel_times(reset=True)
for _ in range(3):
    f.enqueue(b)
kt = f.kernel_times(reset=True)
tot = sum(v[0] for v in kt.values())
for k, (m, n) in kt.items():
    if n:
        print(f"  {k:16s} {m/3:8.3f} ms/iter  {n/3:6.0f} launches/iter  {100*m/tot:5.1f}%")
