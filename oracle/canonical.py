"""TEST INFRASTRUCTURE ONLY: a pure-Python (numpy) restatement of the canonical
hybrid batch's descriptor, so the CPU reference arm of bench.py can build its
input without loading any product library.

The reference's canonical batch (proj/src/sched.cpp:159-169): n_dec decodes at
prefix kv_each (request ids 0..n_dec-1), then one prompt-completing chunk of
tau - n_dec tokens at chunk_prefix (request id n_dec). Entry semantics follow
core.cpp:42-63 (decode = 1 query at position prefix; chunk = positions prefix ..
prefix+chunk-1). Block ids follow the product's ledger allocation order
(KvLedger::grow in entry order from a free list handing out 0, 1, 2, ...), and
token ids follow include/ss_synth.h ss_token_id; tests/test_oracle.py checks this
module against the C++ host descriptor array by array.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

M64 = (1 << 64) - 1
TAG_TOKEN = 0xA0000


def _mix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def token_id(seed: int, rid: int, pos: int, vocab: int) -> int:
    """ss_token_id (include/ss_synth.h): splitmix64 key of (seed, TAG_TOKEN, rid, pos) mod vocab."""
    k = _mix64(seed ^ ((0x9E3779B97F4A7C15 * (TAG_TOKEN + 1)) & M64)) ^ _mix64((rid * 0xD1B54A32D192ED03 + pos) & M64)
    return _mix64(k) % vocab


class BatchDescC(C.Structure):
    """Layout of ss_batch_desc (include/ss_gpu.h)."""
    _fields_ = [
        ("num_entries", C.c_int32), ("num_tokens", C.c_int32), ("cu_q", C.POINTER(C.c_int32)),
        ("ctx_len", C.POINTER(C.c_int32)), ("pos", C.POINTER(C.c_int32)), ("token_ids", C.POINTER(C.c_int32)),
        ("slot", C.POINTER(C.c_int64)), ("block_table", C.POINTER(C.c_int32)), ("max_blocks", C.c_int32),
        ("out_rows", C.POINTER(C.c_int32)), ("n_out", C.c_int32),
    ]


class CanonicalDesc:
    def __init__(self, tau: int, n_dec: int = 32, kv_each: int = 4096, chunk_prefix: int = 0, *,
                 block_size: int = 16, vocab: int, token_seed: int = 0):
        assert tau - n_dec >= 1
        entries = [(r, 1, kv_each) for r in range(n_dec)] + [(n_dec, tau - n_dec, chunk_prefix)]
        tables, nxt = [], 0
        for _, n, pre in entries:
            nb = (pre + n + block_size - 1) // block_size
            tables.append(list(range(nxt, nxt + nb)))
            nxt += nb
        maxb = max(len(t) for t in tables)
        self.pool_blocks = nxt
        bt = np.full((len(entries), maxb), -1, np.int32)
        cu, ctx, pos, tok, slot, out = [0], [], [], [], [], []
        for e, (rid, n, pre) in enumerate(entries):
            bt[e, :len(tables[e])] = tables[e]
            ctx.append(pre + n)
            for j in range(n):
                p = pre + j
                pos.append(p)
                tok.append(token_id(token_seed, rid, p, vocab))
                slot.append(tables[e][p // block_size] * block_size + p % block_size)
            cu.append(len(pos))
            out.append(len(pos) - 1)  # every decode, and the prompt-completing chunk
        self._a = {"cu_q": np.array(cu, np.int32), "ctx_len": np.array(ctx, np.int32),
                   "pos": np.array(pos, np.int32), "token_ids": np.array(tok, np.int32),
                   "slot": np.array(slot, np.int64), "block_table": bt, "out_rows": np.array(out, np.int32)}
        a = self._a
        P = lambda x, t: x.ctypes.data_as(C.POINTER(t))
        self.view = BatchDescC(len(entries), len(pos), P(a["cu_q"], C.c_int32), P(a["ctx_len"], C.c_int32),
                               P(a["pos"], C.c_int32), P(a["token_ids"], C.c_int32), P(a["slot"], C.c_int64),
                               P(a["block_table"], C.c_int32), maxb, P(a["out_rows"], C.c_int32), len(out))

    def arrays(self) -> dict:
        return {k: v.copy() for k, v in self._a.items()}
