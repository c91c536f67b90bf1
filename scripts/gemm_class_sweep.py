"""Per-projection GEMM schedule sweep inside the real forward (dev tool): for each candidate
(mode, BN[, splits]) set SS_GEMM_<class> and report each projection's device time per launch.
usage: gemm_class_sweep.py [model] [tau] [layers]"""
import os, subprocess, sys, json
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
model = sys.argv[1] if len(sys.argv) > 1 else "mistral7b"
tau = sys.argv[2] if len(sys.argv) > 2 else "512"
layers = sys.argv[3] if len(sys.argv) > 3 else "8"
cands = [(0, 256), (0, 128), (0, 192), (0, 224), (3, 256), (3, 192), (3, 128), (3, 224), (2, 256, 2), (2, 256, 4), (2, 128, 2)]
if os.environ.get("CANDS"):
    cands = [tuple(int(v) for v in c.split(",")) for c in os.environ["CANDS"].split(";")]
classes = {"QKV": ("gemm_qkv", 128), "O": ("gemm_o", 32), "GATEUP": ("gemm_gate_up", 64), "DOWN": ("gemm_down", 32),
           "LMHEAD": ("lm_head", 32)}
code = r'''
import sys, os, json
sys.path.insert(0, os.environ["ROOT"])
from paper_2403_02310_b200 import gpu, host
name = sys.argv[1]
if ":" in name:  # model:tp -> one tensor-parallel rank's shard as a TP1 model
    mname, tp = name.split(":")
    tp = int(tp)
    m = gpu.MODELS[mname]
    shape = gpu.ModelShape(f"{mname}_tp{tp}", int(sys.argv[3]), m.hidden, m.num_q_heads // tp, m.num_kv_heads // tp,
                           m.head_dim, m.ffn // tp, m.vocab // tp, rope_theta=m.rope_theta)
else:
    shape = gpu.MODELS[name].with_layers(int(sys.argv[3]))
f = gpu.HybridForward(shape, weight_seed=1234)
if int(sys.argv[2]) == 0:  # decode-only: 32 decodes at 4096
    d = host.Descriptor.build([host.BatchEntry(i, "decode", 1, 4096) for i in range(32)], vocab=shape.vocab)
else:
    d = host.Descriptor.canonical(int(sys.argv[2]), 32, 4096, 0, vocab=shape.vocab)
f.kv_alloc(d.pool_blocks)
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
print(json.dumps({k: v[0] / v[1] * 1e3 for k, v in kt.items() if v[1]}))
'''
res = {}
for c in [None] + cands:
    env = dict(os.environ, ROOT=ROOT)
    tag = "default" if c is None else ",".join(map(str, c))
    if c is not None:
        for cls, (_, mult) in classes.items():
            if c[1] % mult == 0:
                env["SS_GEMM_" + cls] = tag
    out = subprocess.run([sys.executable, "-c", code, model, tau, layers], env=env, capture_output=True, text=True)
    try:
        kt = json.loads(out.stdout.strip().splitlines()[-1])
    except Exception:
        print(tag, "FAILED", out.stderr[-300:], flush=True)
        continue
    row = []
    for cls, (key, mult) in classes.items():
        if c is None or c[1] % mult == 0:
            row.append(f"{cls}={kt.get(key, 0):6.1f}")
        else:
            row.append(f"{cls}=   -  ")
    print(f"{tag:10s} " + "  ".join(row) + f"   attn={kt.get('attention', 0):6.1f} us", flush=True)
