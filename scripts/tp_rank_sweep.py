"""Per-rank compute time of the BASELINE tensor-parallel configurations on ONE B200 (dev
tool): one rank's shard (q/kv heads, ffn and vocab divided by tp) run as a TP1 model over the
canonical batch — the kernels and shapes a real rank runs, without the collectives (the O /
down epilogues add the residual instead of writing a bf16 partial).
usage: tp_rank_sweep.py [steps]"""
import os, sys, time
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import torch
from paper_2403_02310_b200 import gpu, host

CONFIGS = [("yi34b", 2, 512), ("yi34b", 2, 2048), ("yi34b", 4, 512), ("yi34b", 4, 2048),
           ("llama70b", 8, 512), ("llama70b", 8, 1536), ("falcon180b", 8, 2048)]
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
for model, tp, tau in CONFIGS:
    m = gpu.MODELS[model]
    s = gpu.ModelShape(f"{model}_tp{tp}_rank", m.num_layers, m.hidden, m.num_q_heads // tp, m.num_kv_heads // tp,
                       m.head_dim, m.ffn // tp, m.vocab // tp, rope_theta=m.rope_theta)
    f = gpu.HybridForward(s, weight_seed=1234)
    d = host.Descriptor.canonical(tau, 32, 4096, 0, vocab=s.vocab, token_seed=7)
    f.kv_alloc(d.pool_blocks)
    f.fill_descriptor_prefixes(d, seed=5)
    b = f.upload(d)
    st = f.torch_stream()
    for _ in range(3):
        f.enqueue(b)
    f.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        f.enqueue(b)
    e1.record(st)
    f.synchronize()
    ms = e0.elapsed_time(e1) / steps
    print(f"{model} tp{tp} tau={tau}: per-rank compute {ms:.2f} ms/step ({tau / ms * 1e3:.0f} tok/s per TP group, "
          f"collectives excluded; {2 * m.num_layers} all-reduces of {tau * m.hidden * 2 / 1e6:.1f} MB per step)",
          flush=True)
    b.free()
    f.close()
    del f
    torch.cuda.empty_cache()
