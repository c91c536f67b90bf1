"""The fp32 CPU oracle (oracle/liboracle.so) — pinned before it is trusted.

1. HF pin: chunked prefill + decodes over paged KV through the oracle must
   reproduce HF transformers' full-sequence fp32 logits, non-unit RMSNorm gains
   included, at two shapes: the tiny model (hd 64, GQA 2, theta 1e4;
   tests/golden/hf_tiny_logits.npz) and the production head geometry (hd 128,
   GQA 4, theta 5e6, positions past 2048; hf_hd128_gqa4_logits.npz), both made
   by tests/golden/make_hf_golden.py.
2. Tensor parallelism: the Megatron shard math with an explicit all-reduce
   (torch.distributed gloo, world_size 2) equals the unsharded forward.
3. Paged KV: block tables from the host session are honoured (results do
   not depend on which physical blocks a request got).
"""
import os
import sys

import numpy as np
import pytest

from paper_2403_02310_b200 import gpu, host

orc_mod = pytest.importorskip("oracle.forward")
Oracle = orc_mod.Oracle

GOLDEN_DIR = os.path.join(os.path.dirname(__file__), "golden")
GOLD = os.path.join(GOLDEN_DIR, "hf_tiny_logits.npz")
HF_GOLDENS = ["hf_tiny_logits.npz", "hf_hd128_gqa4_logits.npz"]


def golden_shape(g):
    f = lambda k: g["shape_" + k].item()
    return gpu.ModelShape("hf_golden", int(f("num_layers")), int(f("hidden")), int(f("num_q_heads")),
                          int(f("num_kv_heads")), int(f("head_dim")), int(f("ffn")), int(f("vocab")),
                          rope_theta=float(f("rope_theta")), rms_eps=float(f("rms_eps")))


def _replay(orc, g, schedule, seed, s):
    """schedule: list of steps, each a list of (rid, kind, tokens, prefix); returns {(rid,pos): logits}."""
    sess = host.Session(4096, vocab=s.vocab, token_seed=seed)
    prompts = {}
    for step in schedule:
        for rid, kind, n, pre in step:
            if kind == "decode":
                prompts.setdefault(rid, pre)
    got = {}
    for step in schedule:
        ents = [host.BatchEntry(rid, kind, n, pre) for rid, kind, n, pre in step]
        pl = [prompts.get(rid, int(g["seq_lens"][rid])) for rid, *_ in step]
        d = sess.step(ents, pl)
        lg = orc.forward(d)
        a = d.arrays()
        for i, r in enumerate(a["out_rows"]):
            e = int(np.searchsorted(a["cu_q"], r, side="right") - 1)
            got[(step[e][0], int(a["pos"][r]))] = lg[i]
    return got


def _schedule(seq_lens, prompts, chunk=48):
    # stall-free style: decodes first, then chunks of <= `chunk` tokens per request per step
    steps, done = [], {i: 0 for i in range(len(seq_lens))}
    while any(done[i] < seq_lens[i] for i in done):
        step = []
        for i, L in enumerate(seq_lens):
            if prompts[i] <= done[i] < L:
                step.append((i, "decode", 1, done[i]))
                done[i] += 1
        for i, L in enumerate(seq_lens):
            if done[i] < prompts[i]:
                c = min(chunk - 7 * i, prompts[i] - done[i])
                step.append((i, "prefill", c, done[i]))
                done[i] += c
        steps.append(step)
    return steps


@pytest.mark.parametrize("golden", HF_GOLDENS)
def test_oracle_matches_hf_transformers(golden):
    g = np.load(os.path.join(GOLDEN_DIR, golden))
    s = golden_shape(g)
    seq = [int(x) for x in g["seq_lens"]]
    prompts = [seq[0] - 9, seq[1] - 40, seq[2] - 61]
    orc = Oracle(s, weight_seed=int(g["weight_seed"]), num_blocks=4096)
    got = _replay(orc, g, _schedule(seq, prompts, chunk=48 if seq[2] < 1000 else 400), int(g["token_seed"]), s)
    checked = 0
    for i in range(len(seq)):
        # the host token generator must reproduce the HF input ids exactly
        toks = host.Descriptor.build([host.BatchEntry(i, "prefill", seq[i], 0)], vocab=s.vocab,
                                     token_seed=int(g["token_seed"])).arrays()["token_ids"]
        assert np.array_equal(toks, g[f"tokens_{i}"])
        for k, p in enumerate(g[f"pos_{i}"]):
            if (i, int(p)) in got:
                ref = g[f"logits_{i}"][k]
                np.testing.assert_allclose(got[(i, int(p))], ref, rtol=2e-4, atol=2e-4)
                assert got[(i, int(p))].argmax() == ref.argmax()
                checked += 1
    assert checked >= 15


def test_oracle_block_placement_invariance():
    # the same requests placed in different physical blocks give identical results
    s = gpu.MODELS["tiny"]
    ents = [host.BatchEntry(0, "decode", 1, 200), host.BatchEntry(1, "prefill", 60, 40)]
    d1 = host.Descriptor.build(ents, vocab=s.vocab, token_seed=3)
    d2 = host.Descriptor.build(list(reversed(ents)), vocab=s.vocab, token_seed=3)  # different block ids
    outs = []
    for d in (d1, d2):
        o = Oracle(s, weight_seed=5, num_blocks=64)
        a = d.arrays()
        # fill prefixes keyed by the *request id* of each entry
        for e, rid in enumerate([ents[0].request_id, ents[1].request_id] if d is d1 else [1, 0]):
            pre = int(a["pos"][a["cu_q"][e]])
            o.fill_synthetic(a["block_table"][e][:(pre + 15) // 16], rid, pre, 11)
        outs.append(o.forward(d))
    # d1 rows: [decode(0), chunk(1)]; d2 rows: [chunk(1), decode(0)]
    np.testing.assert_allclose(outs[0][0], outs[1][1], rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(outs[0][1], outs[1][0], rtol=1e-5, atol=1e-5)


def _tp_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
    from oracle.forward import Oracle as O
    from paper_2403_02310_b200 import gpu as G, host as H

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    s = G.ModelShape("tp", 2, 256, 8, 4, 64, 512, 512)
    d = H.Descriptor.canonical(160, 8, 300, 40, vocab=s.vocab, token_seed=1)
    o = O(s, tp_rank=rank, tp_size=world, weight_seed=9, num_blocks=d.pool_blocks)

    def ar(buf):
        t = torch.from_numpy(buf)
        dist.all_reduce(t)

    o.set_allreduce(ar)
    o.fill_descriptor_prefixes(d, 4)
    lg = o.forward(d)
    parts = [torch.zeros_like(torch.from_numpy(lg)) for _ in range(world)]
    dist.all_gather(parts, torch.from_numpy(lg))
    if rank == 0:
        q.put(np.concatenate([p.numpy() for p in parts], axis=1))
    dist.destroy_process_group()


def test_oracle_tensor_parallel_gloo():
    import multiprocessing as mp
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_tp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    tp_logits = q.get(timeout=300)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    s = gpu.ModelShape("tp", 2, 256, 8, 4, 64, 512, 512)
    d = host.Descriptor.canonical(160, 8, 300, 40, vocab=s.vocab, token_seed=1)
    o = Oracle(s, weight_seed=9, num_blocks=d.pool_blocks)
    o.fill_descriptor_prefixes(d, 4)
    ref = o.forward(d)
    np.testing.assert_allclose(tp_logits, ref, rtol=1e-4, atol=1e-4)


@pytest.mark.parametrize("tau,n_dec,kv,prefix,vocab", [(512, 32, 4096, 0, 32000), (2048, 32, 4096, 2048, 64000),
                                                       (160, 8, 300, 40, 512)])
def test_canonical_restatement_matches_host(tau, n_dec, kv, prefix, vocab):
    """oracle/canonical.py (the CPU reference arm's input, no product library) builds the
    same descriptor as the C++ host (ssh_desc_canonical), array for array."""
    from oracle.canonical import CanonicalDesc

    a = CanonicalDesc(tau, n_dec, kv, prefix, vocab=vocab, token_seed=7)
    b = host.Descriptor.canonical(tau, n_dec, kv, prefix, vocab=vocab, token_seed=7)
    assert a.pool_blocks == b.pool_blocks
    ea, eb = a.arrays(), b.arrays()
    for k in ("cu_q", "ctx_len", "pos", "token_ids", "slot", "block_table", "out_rows"):
        assert np.array_equal(ea[k], eb[k]), k
