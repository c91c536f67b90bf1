"""The reference's OWN engine driving the B200 forward (compiled).

oracle/_ref/ref_engine_gpu is the reference's src/engine.cpp with the one-line model-step
patch at engine.cpp:227 applied by sed at build time (oracle/Makefile), linked with the
reference's other sources and oracle/ref_engine_gpu.cpp. Its simulate()/summarize() run the
openchat trace with every iteration's time measured on the GPU through ss_forward_hybrid.
The restated engine (host.simulate with gpu=) runs the same trace with the same forward; the
two schedules see slightly different measured times, so their summaries agree closely rather
than bit for bit.
"""
import json
import os
import subprocess

import pytest

torch = pytest.importorskip("torch")

from paper_2403_02310_b200 import gpu, host  # noqa: E402

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(__file__), "..", "oracle", "_ref", "ref_engine_gpu")


@pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/ref_engine_gpu not built (needs the reference tree)")
def test_reference_engine_drives_the_b200_forward():
    s = gpu.MODELS["mistral7b"]
    pool, n, qps, seed, tau = 20000, 24, 4.0, 42, 512
    args = [str(x) for x in (s.num_layers, s.hidden, s.num_q_heads, s.num_kv_heads, s.head_dim, s.ffn, s.vocab,
                             s.rope_theta, "mistral7b", "openchat", qps, n, seed, tau, pool)]
    out = subprocess.run([BIN] + args, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    ref = json.loads(out.stdout.strip().splitlines()[-1])
    assert ref["n_requests"] == n and ref["gpu_steps"] == ref["microbatches"] > 0
    assert 1.0 < ref["mean_step_ms"] < 50.0  # measured B200 forwards, not the A100 cost model

    f = gpu.HybridForward(s, weight_seed=1234)
    f.kv_alloc(pool)
    cfg = host.ReplicaConfig(token_budget=tau, kv_blocks=pool)
    ours = host.simulate(cfg, host.model_preset("mistral7b"), host.make_trace("openchat", qps, n, seed), gpu=f,
                         token_seed=seed, keep_events=False).summarize()
    f.close()
    assert ours["n_requests"] == ref["n_requests"]
    for k in ("tbt_p99_ms", "tbt_median_ms", "throughput_tps"):
        assert ours[k] == pytest.approx(ref[k], rel=0.3), (k, ours[k], ref[k])
