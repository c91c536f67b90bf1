"""End-to-end parity of the B200 hybrid-batch forward with the fp32 CPU oracle.

Inputs are identical by construction: the same host-built descriptor (block
tables, positions, slots, token ids — the same arrays on both sides, and checked
here against an independent numpy restatement of the reference's batch semantics),
the same counter-based weights, RMSNorm gains and synthetic cache
(include/ss_synth.h). The GPU computes in bf16 with fp32 accumulation; the oracle
in fp32 (itself pinned to HF transformers, tests/test_oracle.py).

Stated tolerance (bf16 compute bound), per configuration in TOL: per logit row
    rel-L2(gpu, oracle) <= rel   and   max-abs <= mabs * max|oracle|,
and greedy top-1 agreement >= top1 over the batch's rows (near-tied logits may
flip under bf16 rounding). The bounds are ~3x the errors measured on B200
(DESIGN.md §2 table, profiles/r02/parity_depth.json).
"""
import gzip
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2403_02310_b200 import gpu, host  # noqa: E402

orc_mod = pytest.importorskip("oracle.forward")
pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
LOG = os.environ.get("SS_PARITY_LOG")  # optional JSONL of measured errors (profiles/r02/parity_depth.json)

# label -> (rel-L2, max-abs fraction, top-1 agreement); ~3x the measured error (see module doc)
TOL = {
    "tiny": (8e-3, 1.0e-2, 0.96),           # measured 2.5e-3 / 2.9e-3 / 1.000
    "decode_only": (8e-3, 1.0e-2, 0.96),    # measured 2.5e-3 / 3.4e-3 / 1.000
    "full_width_2l": (7.5e-3, 1.0e-2, 0.96),  # measured 2.3e-3 / 3.1e-3 / 1.000
    "full_depth": (7.5e-3, 9e-3, 0.96),     # measured 2.4e-3 / 2.9e-3 / 1.000 at 8, 32, 60 layers
    "long_prefix": (8e-3, 9e-3, 0.96),      # measured 2.7e-3 / 2.8e-3 / 1.000
    "trace": (9e-3, 1.4e-2, 0.99),          # measured 3.0e-3 / 4.5e-3 / 0.997 over 30,027 rows
    "tp": (8e-3, 1.0e-2, 0.96),             # tensor-parallel groups (test_gpu_tp_*)
}


def errors(g, o):
    rel = np.linalg.norm(g - o, axis=1) / np.maximum(np.linalg.norm(o, axis=1), 1e-12)
    mabs = np.abs(g - o).max(axis=1) / np.maximum(np.abs(o).max(axis=1), 1e-12)
    top1 = float((g.argmax(1) == o.argmax(1)).mean())
    return float(rel.max()), float(mabs.max()), top1


def log(label, **kv):
    if LOG:
        with open(LOG, "a") as f:
            f.write(json.dumps({"case": label, **kv}) + "\n")


def compare(g, o, label, tol="tp"):
    assert g.shape == o.shape, label
    assert np.isfinite(g).all(), label
    rel, mabs, top1 = errors(g, o)
    log(label, rel_l2=rel, max_abs_frac=mabs, top1=top1, rows=int(len(o)))
    r_tol, m_tol, t_tol = TOL[tol]
    assert rel <= r_tol, f"{label}: rel-L2 {rel:.3e} > {r_tol:.1e}"
    assert mabs <= m_tol, f"{label}: max-abs frac {mabs:.3e} > {m_tol:.1e}"
    assert top1 >= t_tol, f"{label}: top-1 agreement {top1:.3f} < {t_tol}"
    return rel, mabs, top1


def run_pair(s, d, prefix_seed=5):
    f = gpu.HybridForward(s, weight_seed=1234)
    f.kv_alloc(d.pool_blocks)
    f.fill_descriptor_prefixes(d, seed=prefix_seed)
    lg, nt, _ = f.forward(d)
    f.close()
    assert (nt == lg.argmax(1)).all()
    o = orc_mod.Oracle(s, weight_seed=1234, num_blocks=d.pool_blocks)
    o.fill_descriptor_prefixes(d, seed=prefix_seed)
    ref = o.forward(d)
    o.close()
    return lg, ref


YI_TP2_RANK = gpu.ModelShape("yi_tp2_rank", 60, 7168, 28, 4, 128, 10240, 32000, rope_theta=5e6)


@pytest.mark.parametrize("tau,chunk_prefix", [(512, 0), (512, 2048), (2048, 0)])
def test_tiny_canonical_batch(tau, chunk_prefix):
    s = gpu.MODELS["tiny"]
    d = host.Descriptor.canonical(tau, 32, 4096, chunk_prefix, vocab=s.vocab, token_seed=7)
    lg, ref = run_pair(s, d)
    compare(lg, ref, f"tiny tau={tau} prefix={chunk_prefix}", "tiny")


@pytest.mark.parametrize("model", ["mistral7b", "yi34b", "falcon180b"])
def test_full_width_two_layers(model):
    """Full-width shapes at truncated depth (2 layers). Yi-34B and Falcon-180B at one TP
    rank's width (TP2: 28 q / 4 kv heads; TP8: 29 q / 1 kv head, hd 64), run as TP1 math."""
    s = gpu.MODELS[model].with_layers(2)
    if model == "falcon180b":
        s = gpu.ModelShape("falcon_tp8_rank", 2, 14848, 29, 1, 64, 7424, 8128)
    if model == "yi34b":
        s = YI_TP2_RANK.with_layers(2)
    d = host.Descriptor.canonical(512, 32, 4096, 0, vocab=s.vocab, token_seed=7)
    lg, ref = run_pair(s, d)
    compare(lg, ref, f"{s.name} L=2 tau=512", "full_width_2l")


@pytest.mark.parametrize("model,layers", [("mistral7b", 8), ("mistral7b", 32), ("yi34b", 60)])
def test_full_depth_canonical(model, layers):
    """The BASELINE configurations at their real depth on the canonical tau=512 batch
    (32 decodes @ 4096 + a 480-token chunk): error growth over 32 / 60 layers."""
    s = gpu.MODELS[model].with_layers(layers) if model == "mistral7b" else YI_TP2_RANK.with_layers(layers)
    d = host.Descriptor.canonical(512, 32, 4096, 0, vocab=s.vocab, token_seed=7)
    lg, ref = run_pair(s, d)
    compare(lg, ref, f"{s.name} L={layers} tau=512", "full_depth")


@pytest.mark.parametrize("model", ["tiny", "mistral7b"])
def test_long_prefix_chunk(model):
    """A chunk at prefix 12288 (arxiv-like long prompts reach ~16k) next to decodes at
    16k contexts: the split-KV prefill tiles and long decode streams."""
    s = gpu.MODELS[model] if model == "tiny" else gpu.MODELS[model].with_layers(2)
    ents = [host.BatchEntry(i, "decode", 1, 16000 + 97 * i) for i in range(8)]
    ents.append(host.BatchEntry(8, "prefill", 504, 12288))
    d = host.Descriptor.build(ents, completes=[True] * 8 + [True], vocab=s.vocab, token_seed=11)
    lg, ref = run_pair(s, d)
    compare(lg, ref, f"{model} chunk 504 @ prefix 12288 + 8 decodes @ 16k", "long_prefix")


# ------------------------------------------------------------------ reference trace replay
def _mix64(x):
    M = (1 << 64) - 1
    x = (x + 0x9E3779B97F4A7C15) & M
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M
    return x ^ (x >> 31)


def token_id(seed, rid, pos, vocab):
    """Independent restatement of ss_token_id (include/ss_synth.h)."""
    M = (1 << 64) - 1
    k = _mix64(seed ^ ((0x9E3779B97F4A7C15 * (0xA0000 + 1)) & M)) ^ _mix64((rid * 0xD1B54A32D192ED03 + pos) & M)
    return _mix64(k) % vocab


def reference_stream():
    """Micro-batches of the reference's own event log (tiny clock, openchat seed 42,
    qps 16, 64 requests, tau 512; tests/golden/make_golden.py): entries per batch,
    plus each request's prompt / output lengths recovered from the same log."""
    batches, prompt, outputs = [], {}, {}
    with gzip.open(os.path.join(GOLDEN, "tiny_qps16.jsonl.gz"), "rt") as f:
        for line in f:
            ev = json.loads(line)
            if ev["ev"] == "batch_start":
                ents = [(e["r"], e["kind"], e["tokens"], e["prefix"]) for e in ev["entries"]]
                batches.append(ents)
                for r, kind, n, _ in ents:
                    if kind == "prefill":
                        prompt[r] = prompt.get(r, 0) + n
            elif ev["ev"] == "token_emit":
                outputs[ev["r"]] = outputs.get(ev["r"], 0) + 1
    return batches, prompt, outputs


def check_descriptor(a, ents, prompt, seed, vocab, tables):
    """Descriptor = the reference's batch semantics (core.cpp:42-63, engine.cpp:211-216):
    positions, context lengths, logit rows, slots through a per-request block table that
    is stable across steps, distinct blocks between live requests, token ids."""
    out = []
    for e, (rid, kind, n, pre) in enumerate(ents):
        q0, q1 = int(a["cu_q"][e]), int(a["cu_q"][e + 1])
        assert q1 - q0 == n
        pos = a["pos"][q0:q1]
        assert np.array_equal(pos, pre + np.arange(n)) and a["ctx_len"][e] == pre + n
        nb = (pre + n + 15) // 16
        bt = [int(b) for b in a["block_table"][e][:nb]]
        old = tables.get(rid, [])
        assert bt[:len(old)] == old, "a request's block table changed under it"
        tables[rid] = bt
        assert np.array_equal(a["slot"][q0:q1], np.array([bt[p // 16] * 16 + p % 16 for p in pos]))
        assert all(int(a["token_ids"][q0 + j]) == token_id(seed, rid, int(p), vocab) for j, p in enumerate(pos))
        if kind == "decode" or pre + n == prompt[rid]:
            out.append(q1 - 1)
    assert np.array_equal(a["out_rows"], np.array(out, dtype=a["out_rows"].dtype))
    live = [b for bt in tables.values() for b in bt]
    assert len(live) == len(set(live)), "two live requests share a KV block"


def test_reference_trace_replay_tiny():
    """BASELINE configs[0] end to end: EVERY micro-batch (2,276) of the reference's own
    64-request trace is executed on the GPU and on the oracle, each with one persistent
    paged KV pool; descriptors are checked bit-exact against the reference's batch
    semantics and every logit row is compared."""
    s = gpu.MODELS["tiny"]
    batches, prompt, outputs = reference_stream()
    assert len(batches) == 2276
    seed = 42
    sess = host.Session(131072, vocab=s.vocab, token_seed=seed)
    f = gpu.HybridForward(s, weight_seed=1234)
    f.kv_alloc(16384)
    o = orc_mod.Oracle(s, weight_seed=1234, num_blocks=16384)
    tables, rows, agree, worst_rel, worst_abs = {}, 0, 0, 0.0, 0.0
    for ents in batches:
        d = sess.step([host.BatchEntry(r, k, n, p) for r, k, n, p in ents], [prompt[r] for r, *_ in ents])
        check_descriptor(d.arrays(), ents, prompt, seed, s.vocab, tables)
        lg, nt, _ = f.forward(d)
        ref = o.forward(d)
        if len(ref):
            rel, mabs, _ = errors(lg, ref)
            worst_rel, worst_abs = max(worst_rel, rel), max(worst_abs, mabs)
            rows += len(ref)
            agree += int((lg.argmax(1) == ref.argmax(1)).sum())
            assert (nt == lg.argmax(1)).all()
        for r, kind, n, p in ents:  # the request's last iteration: release its blocks
            if (kind == "decode" and p == prompt[r] + outputs[r] - 2) or (
                    kind == "prefill" and p + n == prompt[r] and outputs[r] == 1):
                sess.release(r)
                tables.pop(r)
    f.close()
    o.close()
    log("tiny reference trace (2276 micro-batches)", rel_l2=worst_rel, max_abs_frac=worst_abs, top1=agree / rows,
        rows=rows)
    r_tol, m_tol, t_tol = TOL["trace"]
    assert rows == sum(outputs.values())  # one logit row per emitted token
    assert worst_rel <= r_tol and worst_abs <= m_tol, (worst_rel, worst_abs)
    assert agree / rows >= t_tol


def test_closed_loop_engine_on_gpu():
    """The engine's model step is the real forward (engine.cpp:227 seam): a
    short trace runs to completion with measured iteration times; the batch
    stream obeys the stall-free invariants (token budget, chunk cover)."""
    s = gpu.MODELS["tiny"]
    trace = host.make_trace("openchat", 8, 12, 3)
    f = gpu.HybridForward(s, weight_seed=1234)
    f.kv_alloc(20000)
    rep = host.simulate(host.ReplicaConfig(kv_blocks=20000), host.model_preset("tiny"), trace, gpu=f, token_seed=1,
                        check_block_tables=True)
    summ = rep.summarize()
    assert summ["n_requests"] == 12 and summ["tbt_samples"] > 0
    covered = {}
    for mb in rep.microbatches():
        assert mb.total_tokens <= 512
        assert mb.iteration_ms > 0
        for e in mb.entries:
            if e.kind == "prefill":
                assert e.prefix_tokens == covered.get(e.request_id, 0)
                covered[e.request_id] = e.prefix_tokens + e.chunk_tokens
    assert all(covered[i] == r.prompt_tokens for i, r in enumerate(trace))
    f.close()


def test_gpu_executor_rejects_pipeline_and_tp_mismatch():
    """The GPU step is a whole-model forward of this context's TP shard: a pipelined
    replica or another tp degree is a contract violation, not a silently wrong clock."""
    s = gpu.MODELS["tiny"]
    trace = host.make_trace("openchat", 8, 4, 3)
    f = gpu.HybridForward(s, weight_seed=1234)
    f.kv_alloc(4000)
    for cfg in (host.ReplicaConfig(kv_blocks=4000, pp_degree=2), host.ReplicaConfig(kv_blocks=4000, tp_degree=2)):
        with pytest.raises(host.ContractViolation):
            host.simulate(cfg, host.model_preset("tiny"), trace, gpu=f, token_seed=1)
    f.close()


@pytest.mark.parametrize("model,n_dec", [("tiny", 32), ("tiny", 7), ("mistral7b", 24)])
def test_decode_only_batch(model, n_dec):
    """Decode-only iterations (the bulk of a replayed trace): M <= 32 projections run on
    single-CTA tiles that stage only 32 rows of A per stage; parity with the oracle."""
    s = gpu.MODELS[model] if model == "tiny" else gpu.MODELS[model].with_layers(2)
    ents = [host.BatchEntry(i, "decode", 1, 100 + 37 * i) for i in range(n_dec)]
    d = host.Descriptor.build(ents, vocab=s.vocab, token_seed=3)
    lg, ref = run_pair(s, d)
    compare(lg, ref, f"{model} decode-only x{n_dec}", "decode_only")


def test_device_selection_from_another_current_device():
    """ss_create(device=d) allocates everything on d whatever the calling thread's current
    device is (the stream-K workspace included); with one GPU this checks that creation
    works from a thread whose current device was never set."""
    import threading

    res = {}

    def body():
        try:
            f = gpu.HybridForward(gpu.MODELS["tiny"], weight_seed=1234, device=torch.cuda.device_count() - 1)
            d = host.Descriptor.canonical(64, 4, 100, 0, vocab=512, token_seed=1)
            f.kv_alloc(d.pool_blocks)
            lg, nt, _ = f.forward(d)
            res["ok"] = bool(np.isfinite(lg).all())
            f.close()
        except Exception as e:  # pragma: no cover
            res["err"] = repr(e)

    t = threading.Thread(target=body)
    t.start()
    t.join()
    assert res.get("ok"), res
