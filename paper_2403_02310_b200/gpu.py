"""Python handle on the ss_gpu.h boundary (libss_gpu.so).

`HybridForward` is one tensor-parallel rank of the B200 hybrid-batch forward
that replaces the reference's iteration_time() model step (reference
proj/src/costmodel.cpp:39-56 via engine.cpp:227). Everything below is a thin
ctypes layer: all compute runs in the sm_100a kernels of libss_gpu.so, and
construction fails loudly when no B200 is visible (there is no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence, Tuple

import numpy as np

from . import _lib
from ._lib import gpu_lib


@dataclass(frozen=True)
class ModelShape:
    name: str
    num_layers: int
    hidden: int
    num_q_heads: int
    num_kv_heads: int
    head_dim: int
    ffn: int
    vocab: int
    rope_theta: float = 10000.0
    rms_eps: float = 1e-5
    max_positions: int = 16384 + 1024

    def c(self) -> _lib.ModelCfg:
        return _lib.ModelCfg(self.num_layers, self.hidden, self.num_q_heads, self.num_kv_heads, self.head_dim,
                             self.ffn, self.vocab, self.rope_theta, self.rms_eps, self.max_positions)

    def with_layers(self, n: int) -> "ModelShape":
        return ModelShape(self.name, n, self.hidden, self.num_q_heads, self.num_kv_heads, self.head_dim, self.ffn,
                          self.vocab, self.rope_theta, self.rms_eps, self.max_positions)

    def params_per_layer(self) -> int:
        h, hd = self.hidden, self.head_dim
        return h * (self.num_q_heads + 2 * self.num_kv_heads) * hd + self.num_q_heads * hd * h + 3 * h * self.ffn


# Reference carries only hidden/ffn (presets.cpp:8-66); head geometry from the
# public configs. "tiny" is BASELINE.json configs[0].
MODELS = {
    "tiny": ModelShape("tiny", 2, 256, 4, 2, 64, 704, 512, max_positions=16384 + 1024),
    "mistral7b": ModelShape("mistral7b", 32, 4096, 32, 8, 128, 14336, 32000),
    "yi34b": ModelShape("yi34b", 60, 7168, 56, 8, 128, 20480, 64000, rope_theta=5e6),
    "llama70b": ModelShape("llama70b", 80, 8192, 64, 8, 128, 28672, 32000),
    "falcon180b": ModelShape("falcon180b", 80, 14848, 232, 8, 64, 59392, 65024),
}

KERNEL_CLASSES = ["embed", "rmsnorm", "gemm_qkv", "rope_kv_append", "attention", "attn_combine", "gemm_o",
                  "gemm_gate_up", "gemm_down", "nccl_allreduce", "lm_head", "argmax", "gemm_chain"]


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    st = gpu_lib().ss_nccl_unique_id(buf)
    if st:
        _lib.raise_for(st, gpu_lib().ss_last_error(None).decode())
    return bytes(buf)


class _Dev:
    """__cuda_array_interface__ view of library-owned device memory."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"data": (ptr, False), "shape": tuple(shape), "typestr": typestr,
                                         "version": 3, "strides": None}


class Batch:
    def __init__(self, fwd: "HybridForward", handle: int, n_out: int, num_tokens: int):
        self._fwd, self._h, self.n_out, self.num_tokens = fwd, C.c_void_p(handle), n_out, num_tokens

    @property
    def handle(self):
        return self._h

    def free(self):
        if self._h is not None and self._h.value:
            gpu_lib().ss_batch_free(self._fwd._h, self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class HybridForward:
    def __init__(self, shape: ModelShape, tp_rank: int = 0, tp_size: int = 1, nccl_id: Optional[bytes] = None,
                 weight_seed: int = 1234, device: int = 0):
        self.shape = shape
        self.tp_rank, self.tp_size = tp_rank, tp_size
        idbuf = None
        if nccl_id is not None:
            idbuf = (C.c_char * 128).from_buffer_copy(nccl_id)
        h = C.c_void_p()
        st = gpu_lib().ss_create(C.byref(shape.c()), tp_rank, tp_size, idbuf, weight_seed, device, C.byref(h))
        if st:
            _lib.raise_for(st, gpu_lib().ss_last_error(None).decode())
        self._h = h
        self.kv_blocks = 0

    @classmethod
    def _adopt(cls, shape: ModelShape, handle: int, tp_rank: int, tp_size: int) -> "HybridForward":
        self = cls.__new__(cls)
        self.shape, self.tp_rank, self.tp_size = shape, tp_rank, tp_size
        self._h = C.c_void_p(handle)
        self.kv_blocks = 0
        return self

    @property
    def handle(self):
        return self._h

    def ipc_connect(self, allgather, max_tokens: int = 8192):
        """CUDA-IPC TP transport (a rank created without an NCCL id): exports this rank's
        exchange region, all-gathers the 64-byte handles with `allgather(bytes) -> list`
        (rank order, e.g. torch.distributed.all_gather_object) and maps every peer's."""
        buf = (C.c_char * 64)()
        self._check(gpu_lib().ss_ipc_export(self._h, max_tokens, buf))
        handles = allgather(bytes(buf))
        assert len(handles) == self.tp_size and all(len(x) == 64 for x in handles)
        allh = (C.c_char * (64 * self.tp_size)).from_buffer_copy(b"".join(handles))
        self._check(gpu_lib().ss_ipc_open(self._h, allh))

    def _check(self, st: int):
        if st:
            _lib.raise_for(st, gpu_lib().ss_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            gpu_lib().ss_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- KV pool
    def kv_alloc(self, num_blocks: int, block_size: int = 16):
        self._check(gpu_lib().ss_kv_alloc(self._h, num_blocks, block_size))
        self.kv_blocks = num_blocks

    def fill_synthetic(self, block_table: np.ndarray, request_id: int, n_tokens: int, seed: int):
        bt = np.ascontiguousarray(block_table, dtype=np.int32)
        self._check(gpu_lib().ss_kv_fill_synthetic(self._h, bt.ctypes.data, len(bt), request_id, n_tokens, seed))

    def fill_descriptor_prefixes(self, desc, seed: int):
        """Synthetic cache for every entry's cached prefix (positions < pos[first token])."""
        a = desc.arrays()
        for e in range(len(a["ctx_len"])):
            prefix = int(a["pos"][a["cu_q"][e]])
            if prefix > 0:
                nb = (prefix + 15) // 16
                self.fill_synthetic(a["block_table"][e][:nb], e, prefix, seed)

    # ---- forward
    def forward(self, desc, logits: bool = True) -> Tuple[Optional[np.ndarray], np.ndarray, float]:
        """ss_forward_hybrid from host descriptor arrays; returns (logits, next tokens, device ms)."""
        v = desc.view if hasattr(desc, "view") else desc
        n_out = v.n_out
        lg = np.empty((n_out, self.shape.vocab), np.float32) if logits else None
        nt = np.empty(n_out, np.int32)
        ms = C.c_float()
        self._check(gpu_lib().ss_forward_hybrid(self._h, C.byref(v), lg.ctypes.data if logits else None,
                                                nt.ctypes.data, C.byref(ms)))
        return lg, nt, ms.value

    def upload(self, desc) -> Batch:
        v = desc.view if hasattr(desc, "view") else desc
        b = C.c_void_p()
        self._check(gpu_lib().ss_batch_upload(self._h, C.byref(v), C.byref(b)))
        return Batch(self, b.value, v.n_out, v.num_tokens)

    def enqueue(self, batch: Batch):
        self._check(gpu_lib().ss_forward_enqueue(self._h, batch.handle))

    def read_outputs(self, batch: Batch, logits: bool = False):
        lg = np.empty((batch.n_out, self.shape.vocab), np.float32) if logits else None
        nt = np.empty(batch.n_out, np.int32)
        self._check(gpu_lib().ss_read_outputs(self._h, batch.handle, lg.ctypes.data if logits else None,
                                              nt.ctypes.data))
        return lg, nt

    def synchronize(self):
        self._check(gpu_lib().ss_synchronize(self._h))

    @property
    def stream_ptr(self) -> int:
        return gpu_lib().ss_stream(self._h)

    def torch_stream(self):
        import torch

        return torch.cuda.ExternalStream(self.stream_ptr)

    # ---- TP all-reduce algorithm of the IPC transport (ss_set_tp_allreduce)
    ALLREDUCE = {"auto": 0, "oneshot": 1, "twoshot": 2, "push": 3}

    def set_tp_allreduce(self, algo: str):
        self._check(gpu_lib().ss_set_tp_allreduce(self._h, self.ALLREDUCE[algo]))

    # ---- CUDA graphs of the forward (one per batch shape; ss_set_graphs)
    def set_graphs(self, on: bool):
        self._check(gpu_lib().ss_set_graphs(self._h, int(on)))

    def graph_stats(self) -> Tuple[int, int]:
        """(graphs captured, graph replays) since creation."""
        cap, rep = C.c_int64(), C.c_int64()
        self._check(gpu_lib().ss_graph_stats(self._h, C.byref(cap), C.byref(rep)))
        return cap.value, rep.value

    # ---- profiling
    def set_profiling(self, on: bool):
        self._check(gpu_lib().ss_set_profiling(self._h, int(on)))

    def kernel_times(self, reset: bool = True) -> dict:
        ms = (C.c_double * len(KERNEL_CLASSES))()
        n = (C.c_int64 * len(KERNEL_CLASSES))()
        self._check(gpu_lib().ss_kernel_times(self._h, ms, n, int(reset)))
        return {k: (ms[i], n[i]) for i, k in enumerate(KERNEL_CLASSES)}

    @property
    def launch_count(self) -> int:
        return gpu_lib().ss_launch_count(self._h)

    # ---- raw views for the per-kernel tests
    def weight(self, name: str, layer: int = 0):
        import torch

        p, r, c = C.c_void_p(), C.c_int64(), C.c_int64()
        self._check(gpu_lib().ss_weight_ptr(self._h, name.encode(), layer, C.byref(p), C.byref(r), C.byref(c)))
        return torch.as_tensor(_Dev(p.value, (r.value, c.value), "<i2"), device="cuda").view(torch.bfloat16)

    def kv_layer(self, layer: int):
        """Raw views [blocks][kv heads][16][hd] of layer `layer`'s K and V pools. Each
        (block, head) page is stored pre-swizzled (the shared-memory image of a SWIZZLE_128B
        box, csrc/gpu/common.cuh kv_page_elem): read values through kv_logical()."""
        import torch

        k, v = C.c_void_p(), C.c_void_p()
        self._check(gpu_lib().ss_kv_layer_ptrs(self._h, layer, C.byref(k), C.byref(v)))
        s = self.shape
        shp = (self.kv_blocks, s.num_kv_heads // self.tp_size, 16, s.head_dim)
        mk = lambda p: torch.as_tensor(_Dev(p, shp, "<i2"), device="cuda").view(torch.bfloat16)
        return mk(k.value), mk(v.value)

    # The single-kernel entry points run on the library stream; torch work that
    # produced their inputs runs on torch's stream, so order the two explicitly.
    @staticmethod
    def _fence():
        import torch

        torch.cuda.synchronize()

    def k_gemm(self, A, B, D, M: int, N: int, K: int, epilogue: int):
        self._fence()
        self._check(gpu_lib().ss_k_gemm(self._h, A.data_ptr(), B.data_ptr(), D.data_ptr(), M, N, K, epilogue))

    def k_rmsnorm(self, x, w, out, rows, M: int, h: int, eps: float):
        self._fence()
        self._check(gpu_lib().ss_k_rmsnorm(self._h, x.data_ptr(), w.data_ptr(), out.data_ptr(),
                                           rows.data_ptr() if rows is not None else None, M, h, eps))

    def k_rope_append(self, qkv, q_out, pos, slot, T: int, layer: int):
        self._fence()
        self._check(gpu_lib().ss_k_rope_append(self._h, qkv.data_ptr(), q_out.data_ptr(), pos.data_ptr(),
                                               slot.data_ptr(), T, layer))

    def k_attention(self, batch: Batch, q, o, layer: int):
        self._fence()
        self._check(gpu_lib().ss_k_attention(self._h, batch.handle, q.data_ptr(), o.data_ptr(), layer))


class LocalTPGroup:
    """tp rank contexts on ONE device (ss_create_local_group): the sharded forward
    of a tp-GPU job with NCCL replaced by barriers + peer-sum kernels, so tensor
    parallelism can be checked against the oracle where one GPU is visible."""

    def __init__(self, shape: ModelShape, tp_size: int, weight_seed: int = 1234, device: int = 0):
        self.shape, self.tp_size = shape, tp_size
        hs = (C.c_void_p * tp_size)()
        st = gpu_lib().ss_create_local_group(C.byref(shape.c()), tp_size, weight_seed, device, hs)
        if st:
            _lib.raise_for(st, gpu_lib().ss_last_error(None).decode())
        self._hs = hs
        self.ranks = [HybridForward._adopt(shape, hs[r], r, tp_size) for r in range(tp_size)]

    def kv_alloc(self, num_blocks: int, block_size: int = 16):
        for r in self.ranks:
            r.kv_alloc(num_blocks, block_size)

    def fill_descriptor_prefixes(self, desc, seed: int):
        for r in self.ranks:
            r.fill_descriptor_prefixes(desc, seed)

    def forward(self, desc, logits: bool = True) -> Tuple[Optional[np.ndarray], np.ndarray, float]:
        v = desc.view if hasattr(desc, "view") else desc
        lg = np.empty((v.n_out, self.shape.vocab), np.float32) if logits else None
        nt = np.empty(v.n_out, np.int32)
        ms = C.c_float()
        st = gpu_lib().ss_forward_local_group(self._hs, self.tp_size, C.byref(v), lg.ctypes.data if logits else None,
                                              nt.ctypes.data, C.byref(ms))
        self.ranks[0]._check(st)
        return lg, nt, ms.value

    def close(self):
        for r in self.ranks:
            r.close()


class PipelineGroup:
    """Pipeline-parallel stages (ss_create_pp_stage): stage s holds layers
    [s*L/pp, (s+1)*L/pp) (the reference's even split, engine.cpp:42-81), the
    embedding on stage 0 and the LM head on the last; the residual stream is handed
    from stage to stage (a peer copy when the stages sit on different devices).
    `devices` places the stages (default: all on `device`)."""

    def __init__(self, shape: ModelShape, pp: int, weight_seed: int = 1234, device: int = 0,
                 devices: Optional[Sequence[int]] = None):
        self.shape, self.pp = shape, pp
        devices = list(devices) if devices is not None else [device] * pp
        assert len(devices) == pp
        hs = (C.c_void_p * pp)()
        self.stages = []
        for s in range(pp):
            h = C.c_void_p()
            st = gpu_lib().ss_create_pp_stage(C.byref(shape.c()), s, pp, weight_seed, devices[s], C.byref(h))
            if st:
                for x in self.stages:
                    x.close()
                _lib.raise_for(st, gpu_lib().ss_last_error(None).decode())
            hs[s] = h.value
            self.stages.append(HybridForward._adopt(shape, h.value, 0, 1))
        self._hs = hs
        self.stage_ms = [0.0] * pp

    @property
    def handles(self):
        return self._hs

    def kv_alloc(self, num_blocks: int, block_size: int = 16):
        for s in self.stages:
            s.kv_alloc(num_blocks, block_size)

    def fill_descriptor_prefixes(self, desc, seed: int):
        for s in self.stages:
            s.fill_descriptor_prefixes(desc, seed)

    def forward(self, desc, logits: bool = True) -> Tuple[Optional[np.ndarray], np.ndarray, float]:
        """ss_forward_pipeline; returns (logits, next tokens, slowest stage's device ms);
        every stage's time is left in self.stage_ms."""
        v = desc.view if hasattr(desc, "view") else desc
        lg = np.empty((v.n_out, self.shape.vocab), np.float32) if logits else None
        nt = np.empty(v.n_out, np.int32)
        ms = (C.c_float * self.pp)()
        st = gpu_lib().ss_forward_pipeline(self._hs, self.pp, C.byref(v), lg.ctypes.data if logits else None,
                                           nt.ctypes.data, ms)
        self.stages[-1]._check(st)
        self.stage_ms = [float(x) for x in ms]
        return lg, nt, max(self.stage_ms)

    def close(self):
        for s in self.stages:
            s.close()


def kv_page_index(hd: int):
    """[16][hd] flat element offsets of (row, column) inside one pre-swizzled K/V page
    (csrc/gpu/common.cuh kv_page_elem)."""
    import torch

    r = torch.arange(16).view(16, 1)
    d = torch.arange(hd).view(1, hd)
    return (d // 64) * 1024 + r * 64 + ((((d % 64) // 8) ^ (r % 8)) * 8) + d % 8


def kv_logical(pages):
    """Logical [..., 16, hd] values of pre-swizzled pages (a kv_layer view or a slice of one)."""
    idx = kv_page_index(pages.shape[-1]).to(pages.device).reshape(-1)
    flat = pages.reshape(*pages.shape[:-2], -1)
    return flat[..., idx].reshape(pages.shape)
