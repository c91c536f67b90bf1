"""TEST INFRASTRUCTURE ONLY: ctypes driver of liboracle.so, the fp32 CPU
restatement of the hybrid-batch forward (see oracle/oracle.h). Only tests/,
__graft_entry__.smoke() and bench.py's CPU legs may import this module.

Self-contained: it loads no product library (the struct layouts below mirror
include/ss_gpu.h), so bench.py's CPU reference arm maps only liboracle.so."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
AR_FN = C.CFUNCTYPE(None, C.POINTER(C.c_float), C.c_int64, C.c_void_p)

_L = None


class ModelCfgC(C.Structure):
    """Layout of ss_model_cfg (include/ss_gpu.h)."""
    _fields_ = [
        ("num_layers", C.c_int32), ("hidden", C.c_int32), ("num_q_heads", C.c_int32),
        ("num_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("ffn", C.c_int32), ("vocab", C.c_int32),
        ("rope_theta", C.c_float), ("rms_eps", C.c_float), ("max_positions", C.c_int32),
    ]


def model_cfg(shape) -> ModelCfgC:
    return ModelCfgC(shape.num_layers, shape.hidden, shape.num_q_heads, shape.num_kv_heads, shape.head_dim,
                     shape.ffn, shape.vocab, shape.rope_theta, shape.rms_eps, shape.max_positions)


def lib():
    global _L
    if _L is None:
        if not os.path.exists(ORACLE_SO):
            raise ImportError(f"{ORACLE_SO} missing: run `make -C oracle`")
        L = C.CDLL(ORACLE_SO)
        P = C.c_void_p
        L.orc_create.argtypes = [C.POINTER(ModelCfgC), C.c_int32, C.c_int32, C.c_uint64, C.c_int64, C.c_int32,
                                 C.c_int32]
        L.orc_create.restype = P
        L.orc_destroy.argtypes = [P]
        L.orc_set_allreduce.argtypes = [P, AR_FN, P]
        L.orc_threads.restype = C.c_int32
        L.orc_kv_fill_synthetic.argtypes = [P, P, C.c_int32, C.c_int32, C.c_int32, C.c_uint64]
        L.orc_kv_fill_synthetic.restype = C.c_int32
        L.orc_forward.argtypes = [P, P, P, P]  # ss_batch_desc* (any ctypes struct of that layout)
        L.orc_forward.restype = C.c_int32
        L.orc_weight.argtypes = [P, C.c_char_p, C.c_int32, P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.orc_weight.restype = C.c_int32
        L.orc_last_error.restype = C.c_char_p
        _L = L
    return _L


class Oracle:
    def __init__(self, shape, tp_rank=0, tp_size=1, weight_seed=1234, num_blocks=1024, layers=None, with_head=True):
        self.shape, self.tp_rank, self.tp_size = shape, tp_rank, tp_size
        n = shape.num_layers if layers is None else layers
        self._h = lib().orc_create(C.byref(model_cfg(shape)), tp_rank, tp_size, weight_seed, num_blocks, n,
                                   int(with_head))
        if not self._h:
            raise RuntimeError(lib().orc_last_error().decode())
        self._ar = None

    def close(self):
        if self._h:
            lib().orc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_allreduce(self, fn):
        """fn(np.ndarray float32 view) reduces in place across the TP group."""
        def cb(ptr, n, _user):
            fn(np.ctypeslib.as_array(ptr, shape=(n,)))
        self._ar = AR_FN(cb)
        lib().orc_set_allreduce(self._h, self._ar, None)

    def fill_synthetic(self, block_table, rid, n_tokens, seed):
        bt = np.ascontiguousarray(block_table, dtype=np.int32)
        if lib().orc_kv_fill_synthetic(self._h, bt.ctypes.data, len(bt), rid, n_tokens, seed):
            raise RuntimeError("bad synthetic fill")

    def fill_descriptor_prefixes(self, desc, seed):
        a = desc.arrays()
        for e in range(len(a["ctx_len"])):
            prefix = int(a["pos"][a["cu_q"][e]])
            if prefix > 0:
                self.fill_synthetic(a["block_table"][e][:(prefix + 15) // 16], e, prefix, seed)

    def forward(self, desc, want_hidden=False):
        v = desc.view if hasattr(desc, "view") else desc
        vl = self.shape.vocab // self.tp_size
        lg = np.zeros((v.n_out, vl), np.float32)
        hid = np.zeros((v.num_tokens, self.shape.hidden), np.float32) if want_hidden else None
        st = lib().orc_forward(self._h, C.addressof(v), lg.ctypes.data, hid.ctypes.data if want_hidden else None)
        if st:
            raise RuntimeError(lib().orc_last_error().decode())
        return (lg, hid) if want_hidden else lg

    def weight(self, name, layer=0):
        r, c = C.c_int64(), C.c_int64()
        if lib().orc_weight(self._h, name.encode(), layer, None, C.byref(r), C.byref(c)):
            raise KeyError(name)
        out = np.empty((r.value, c.value), np.float32)
        lib().orc_weight(self._h, name.encode(), layer, out.ctypes.data, None, None)
        return out


def threads() -> int:
    return lib().orc_threads()
