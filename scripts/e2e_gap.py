"""Where the end-to-end (host descriptor -> next tokens) time goes beyond the device time
(dev tool): per ss_forward_hybrid call, the host phases (ss_debug_host_times) and the device
elapsed time, for the canonical batch with CUDA graphs on and off."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import numpy as np

from paper_2403_02310_b200 import gpu, host

MODEL = os.environ.get("MODEL", "mistral7b")
shape = gpu.MODELS[MODEL]
lib = gpu.gpu_lib()
lib.ss_debug_host_times.restype = C.c_int
lib.ss_debug_host_times.argtypes = [C.c_void_p, C.c_void_p]
f = gpu.HybridForward(shape, weight_seed=1234)
d = host.Descriptor.canonical(512, 32, 4096, 0, vocab=shape.vocab, token_seed=1)
f.kv_alloc(d.pool_blocks)
f.fill_descriptor_prefixes(d, seed=5)
view = d.view
for graphs in (True, False):
    f.set_graphs(graphs)
    for _ in range(4):
        f.forward(view, logits=False)
    rows = []
    ht = np.zeros(3)
    for _ in range(30):
        t0 = time.perf_counter()
        _, _, ms = f.forward(view, logits=False)
        wall = (time.perf_counter() - t0) * 1e3
        assert lib.ss_debug_host_times(f._h, ht.ctypes.data) == 0
        rows.append((wall, ms, *ht))
    r = np.median(np.array(rows), axis=0)
    print(f"graphs {'on ' if graphs else 'off'}: wall {r[0]:.3f} ms, device(ev0..ev1) {r[1]:.3f} ms, "
          f"host prep {r[2]:.1f} us, enqueue {r[3]:.1f} us, D2H+wait {r[4]:.1f} us, "
          f"python+ctypes {r[0] * 1e3 - r[2] - r[3] - r[4]:.1f} us")
