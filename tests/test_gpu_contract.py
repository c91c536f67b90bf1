"""The C-ABI's error behaviour on malformed batch descriptors, and the smallest batches.

ss_forward_hybrid re-validates every descriptor it is handed (entry token counts and context
lengths, cu_q, positions, slots against the block tables, token ids against the vocabulary,
logit rows; ctx.cu validate()) and returns SS_INVALID_ARG with a message instead of launching
on inconsistent indices. A rejected call leaves the context usable: the next valid forward
gives bitwise the logits of a fresh context. The smallest batches (one decode token, a one-token
chunk at prefix 0, a single long-context decode, a chunk starting on a block boundary) match
the fp32 oracle.
"""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2403_02310_b200 import _lib, gpu, host  # noqa: E402

orc_mod = pytest.importorskip("oracle.forward")
from test_gpu_forward import compare, run_pair  # noqa: E402

pytestmark = pytest.mark.gpu

TINY = gpu.MODELS["tiny"]


def make_view(a):
    """A BatchDesc over numpy arrays (kept alive on the returned object)."""
    a = {k: np.ascontiguousarray(v) for k, v in a.items()}
    v = _lib.BatchDesc()
    v.num_entries = len(a["ctx_len"])
    v.num_tokens = len(a["pos"])
    p32 = lambda x: x.ctypes.data_as(C.POINTER(C.c_int32))
    v.cu_q, v.ctx_len, v.pos, v.token_ids = p32(a["cu_q"]), p32(a["ctx_len"]), p32(a["pos"]), p32(a["token_ids"])
    v.slot = a["slot"].ctypes.data_as(C.POINTER(C.c_int64))
    v.block_table = p32(a["block_table"])
    v.max_blocks = a["block_table"].shape[1]
    v.out_rows = p32(a["out_rows"])
    v.n_out = len(a["out_rows"])
    v._keep = a
    return v


def _tamper(a, what):
    a = {k: v.copy() for k, v in a.items()}
    t = int(a["cu_q"][1]) - 1  # last token of entry 0
    if what == "token_id":
        a["token_ids"][t] = TINY.vocab
    elif what == "negative_token_id":
        a["token_ids"][0] = -1
    elif what == "slot":
        a["slot"][t] += 1
    elif what == "pos":
        a["pos"][t] += 1
    elif what == "cu_q":
        a["cu_q"][-1] -= 1
    elif what == "out_rows":
        a["out_rows"][0] = len(a["pos"])
    elif what == "ctx_len":
        a["ctx_len"][0] = 0
    elif what == "ctx_too_long":
        a["ctx_len"][0] = 16 * a["block_table"].shape[1] + 1
    elif what == "block_id":
        a["block_table"][0][0] = 1 << 20
    return a


MESSAGES = {
    "token_id": "token id outside the vocabulary",
    "negative_token_id": "token id outside the vocabulary",
    "slot": "slot disagrees with the block table",
    "pos": "positions must be",
    "cu_q": "cu_q",
    "out_rows": "bad out_rows",
    "ctx_len": "entry with no tokens",
    "ctx_too_long": "context longer than block table",
    "block_id": "outside the KV pool",  # SS_OUT_OF_KV
}


def test_malformed_descriptors_rejected_and_context_survives():
    d = host.Descriptor.canonical(64, 4, 100, 0, vocab=TINY.vocab, token_seed=3)
    a = d.arrays()
    f = gpu.HybridForward(TINY, weight_seed=1234)
    f.kv_alloc(d.pool_blocks)
    f.fill_descriptor_prefixes(d, seed=5)
    lg0, nt0, _ = f.forward(make_view(a))  # the helper's view equals the host's
    lg1, nt1, _ = f.forward(d)
    assert np.array_equal(lg0, lg1) and np.array_equal(nt0, nt1)
    for what, msg in MESSAGES.items():
        with pytest.raises(_lib.SSError) as ei:
            f.forward(make_view(_tamper(a, what)))
        want = 2 if what == "block_id" else 1  # SS_OUT_OF_KV, SS_INVALID_ARG
        assert ei.value.status == want and msg in str(ei.value), (what, str(ei.value))
    lg2, nt2, _ = f.forward(d)
    assert np.array_equal(lg0, lg2) and np.array_equal(nt0, nt2), "a rejected call changed the context"
    f.close()


@pytest.mark.parametrize("ents", [
    [host.BatchEntry(0, "decode", 1, 1)],        # one token over one cached token
    [host.BatchEntry(0, "prefill", 1, 0)],       # a one-token chunk at prefix 0
    [host.BatchEntry(0, "decode", 1, 3000)],     # one long-context decode
    [host.BatchEntry(0, "prefill", 17, 16), host.BatchEntry(1, "decode", 1, 33)],  # ragged: block-boundary prefix
], ids=["decode_ctx1", "prefill_1tok", "decode_ctx3000", "chunk17_at16_plus_decode"])
def test_smallest_batches(ents):
    d = host.Descriptor.build(ents, vocab=TINY.vocab, token_seed=9)
    lg, ref = run_pair(TINY, d)
    compare(lg, ref, f"tiny {d.view.num_tokens}-token batch", "decode_only")
