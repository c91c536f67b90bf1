"""Tensor-parallel forward on one device (ss_create_local_group).

The round's GPU boxes expose one B200, so the tp-GPU job is checked through the
local-group transport: tp rank contexts on the same device, one host thread per
rank, each running the sharded forward (head / column / vocab shards, partial
O and down projections, all-reduce -> residual add, vocab all-gather -> argmax)
exactly as under NCCL, with the collectives done by host barriers and a
peer-sum kernel. Parity is against the fp32 oracle at TP1 (the unsharded math)
with test_gpu_forward's stated tolerance, or, for Falcon-180B's TP8 split where
the oracle at full width would take minutes, against the oracle-checked GPU TP1
path of the same truncated model.
"""
import numpy as np
import pytest

pytest.importorskip("torch")

from paper_2403_02310_b200 import gpu, host  # noqa: E402

orc_mod = pytest.importorskip("oracle.forward")
from test_gpu_forward import compare  # noqa: E402

pytestmark = pytest.mark.gpu

TINY_TP = gpu.ModelShape("tiny_tp", 2, 256, 8, 4, 64, 1024, 512)


def _run_group(shape, tp, d, seed=5):
    g = gpu.LocalTPGroup(shape, tp, weight_seed=1234)
    try:
        g.kv_alloc(d.pool_blocks)
        g.fill_descriptor_prefixes(d, seed=seed)
        lg, nt, ms = g.forward(d)
        lg2, _, _ = g.forward(d)  # re-run: collectives and workspaces are reusable
    finally:
        g.close()
    assert np.array_equal(lg, lg2), "local-group forward is not deterministic"
    assert (nt == lg.argmax(1)).all()
    return lg


def _oracle(shape, d, seed=5):
    o = orc_mod.Oracle(shape, weight_seed=1234, num_blocks=d.pool_blocks)
    o.fill_descriptor_prefixes(d, seed=seed)
    return o.forward(d)


@pytest.mark.parametrize("tp", [2, 4])
@pytest.mark.parametrize("tau,chunk_prefix", [(512, 0), (512, 2048)])
def test_tiny_tp_vs_oracle(tp, tau, chunk_prefix):
    d = host.Descriptor.canonical(tau, 32, 4096, chunk_prefix, vocab=TINY_TP.vocab, token_seed=7)
    compare(_run_group(TINY_TP, tp, d), _oracle(TINY_TP, d), f"tiny tp{tp} tau={tau} prefix={chunk_prefix}")


def test_mistral_tp2_two_layers_vs_oracle():
    s = gpu.MODELS["mistral7b"].with_layers(2)
    d = host.Descriptor.canonical(512, 32, 4096, 0, vocab=s.vocab, token_seed=7)
    compare(_run_group(s, 2, d), _oracle(s, d), "mistral tp2")


def test_yi_tp2_two_layers_vs_oracle():
    """BASELINE.json's Yi-34B TP2 split (28 q / 4 kv heads, ffn 10240, vocab 32000 per rank)."""
    s = gpu.MODELS["yi34b"].with_layers(2)
    d = host.Descriptor.canonical(512, 32, 4096, 0, vocab=s.vocab, token_seed=7)
    compare(_run_group(s, 2, d), _oracle(s, d), "yi34b tp2")


def test_falcon_tp8_two_layers_vs_tp1():
    """Falcon-180B's TP8 split (29 q heads, 1 kv head per rank) vs the GPU TP1 path."""
    s = gpu.MODELS["falcon180b"].with_layers(2)
    d = host.Descriptor.canonical(512, 32, 4096, 0, vocab=s.vocab, token_seed=7)
    lg8 = _run_group(s, 8, d)
    f = gpu.HybridForward(s, weight_seed=1234)
    try:
        f.kv_alloc(d.pool_blocks)
        f.fill_descriptor_prefixes(d, seed=5)
        lg1, _, _ = f.forward(d)
    finally:
        f.close()
    compare(lg8, lg1, "falcon tp8 vs tp1")


def test_group_rejects_partial_rank_list():
    g = gpu.LocalTPGroup(TINY_TP, 2, weight_seed=1)
    try:
        import ctypes as C
        d = host.Descriptor.canonical(512, 4, 256, 0, vocab=TINY_TP.vocab, token_seed=1)
        one = (C.c_void_p * 1)(g._hs[0])
        st = gpu.gpu_lib().ss_forward_local_group(one, 1, C.byref(d.view), None, None, None)
        assert st != 0
    finally:
        g.close()
