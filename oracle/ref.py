"""TEST INFRASTRUCTURE ONLY: ctypes driver of the compiled reference simulator
(oracle/_ref/libservesim_ref.so, built by oracle/Makefile from the reference's
own sources). Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may
import this module.
"""
from __future__ import annotations

import ctypes as C
import os

from paper_2403_02310_b200 import _lib

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libservesim_ref.so")

_ref = None


def available() -> bool:
    return os.path.exists(REF_SO)


def lib():
    global _ref
    if _ref is None:
        if not available():
            raise ImportError(f"{REF_SO} missing (reference tree absent when oracle/ was built)")
        L = C.CDLL(REF_SO)
        P, I32, D = C.c_void_p, C.c_int32, C.c_double
        L.ref_cost_preset.argtypes = [C.c_char_p, C.POINTER(_lib.CostParams)]
        L.ref_cost_preset.restype = I32
        L.ref_make_trace.argtypes = [C.c_char_p, D, I32, C.c_uint64, C.POINTER(_lib.TraceRow)]
        L.ref_make_trace.restype = I32
        L.ref_simulate.argtypes = [C.POINTER(_lib.ReplicaCfg), C.POINTER(_lib.CostParams), C.POINTER(_lib.TraceRow), I32,
                                   C.POINTER(P)]
        L.ref_simulate.restype = I32
        L.ref_report_event_log.argtypes = [P, C.POINTER(C.c_size_t)]
        L.ref_report_event_log.restype = C.c_void_p
        L.ref_summary.argtypes = [P, D, C.POINTER(_lib.Latency)]
        L.ref_summary.restype = I32
        L.ref_report_free.argtypes = [P]
        L.ref_report_free.restype = None
        L.ref_iteration_time.argtypes = [C.POINTER(_lib.EntryRow), I32, C.POINTER(_lib.CostParams), I32, I32]
        L.ref_iteration_time.restype = D
        L.ref_token_budget.argtypes = [D, C.POINTER(_lib.CostParams), I32, C.POINTER(I32)]
        L.ref_token_budget.restype = I32
        L.ref_decode_reference_time.argtypes = [C.POINTER(_lib.CostParams)]
        L.ref_decode_reference_time.restype = D
        L.ref_calibrate.argtypes = [C.POINTER(_lib.AnchorRow), I32, C.POINTER(_lib.CalibOpts), C.POINTER(_lib.CostParams),
                                    C.POINTER(D), C.POINTER(D), C.POINTER(I32)]
        L.ref_calibrate.restype = I32
        L.ref_capacity.argtypes = [C.POINTER(_lib.ReplicaCfg), C.POINTER(_lib.CostParams), C.c_char_p, I32, C.c_uint64,
                                   D, C.POINTER(_lib.CapacityOpts), C.POINTER(D), C.POINTER(I32), P, I32, C.POINTER(I32)]
        L.ref_capacity.restype = I32
        L.ref_last_error.argtypes = []
        L.ref_last_error.restype = C.c_char_p
        _ref = L
    return _ref


def cost_preset(name: str) -> _lib.CostParams:
    c = _lib.CostParams()
    if lib().ref_cost_preset(name.encode(), C.byref(c)) != 0:
        raise KeyError(name)
    return c


def make_trace(workload: str, qps: float, n: int, seed: int):
    arr = (_lib.TraceRow * max(1, n))()
    st = lib().ref_make_trace(workload.encode(), qps, n, seed, arr)
    if st:
        raise RuntimeError(lib().ref_last_error().decode())
    return [(arr[i].arrival_us, arr[i].prompt_tokens, arr[i].output_tokens) for i in range(n)]


def simulate(cfg: _lib.ReplicaCfg, params: _lib.CostParams, trace, warmup: float = 0.05):
    """Returns (status, jsonl, summary dict) of the reference run."""
    arr = (_lib.TraceRow * max(1, len(trace)))()
    for i, (a, p, o) in enumerate(trace):
        arr[i] = _lib.TraceRow(a, p, o)
    h = C.c_void_p()
    st = lib().ref_simulate(C.byref(cfg), C.byref(params), arr, len(trace), C.byref(h))
    if st:
        return st, None, None
    n = C.c_size_t()
    p = lib().ref_report_event_log(h, C.byref(n))
    jsonl = C.string_at(p, n.value).decode()
    lat = _lib.Latency()
    lib().ref_summary(h, warmup, C.byref(lat))
    lib().ref_report_free(h)
    return 0, jsonl, lat.as_dict()


def iteration_time(entries, params: _lib.CostParams, tp: int = 1, pp: int = 1) -> float:
    arr = (_lib.EntryRow * max(1, len(entries)))(*entries)
    return lib().ref_iteration_time(arr, len(entries), C.byref(params), tp, pp)


def token_budget(t_max_ms: float, params: _lib.CostParams, pp: int):
    out = C.c_int32()
    st = lib().ref_token_budget(t_max_ms, C.byref(params), pp, C.byref(out))
    return st, out.value


def decode_reference_time(params: _lib.CostParams) -> float:
    return lib().ref_decode_reference_time(C.byref(params))


def calibrate(anchor_rows, n: int, opts: _lib.CalibOpts):
    """The reference's servesim::calibrate on ssh_anchor rows: (status, params, predicted, max_rel, zeroed_mask)."""
    out = _lib.CostParams()
    pred = (C.c_double * max(1, n))()
    mx = C.c_double()
    mask = C.c_int32()
    st = lib().ref_calibrate(anchor_rows, n, C.byref(opts), C.byref(out), pred, C.byref(mx), C.byref(mask))
    return st, out, list(pred[:n]), mx.value, mask.value


def capacity(cfg: _lib.ReplicaCfg, params: _lib.CostParams, workload: str, n: int, seed: int, slo_ms: float,
             opts: _lib.CapacityOpts):
    """The reference's capacity_search with the CLI probe: (status, qps, monotone, probes)."""
    qps = C.c_double()
    mono = C.c_int32()
    cap = 256
    probes = (_lib.CapacityProbe * cap)()
    npr = C.c_int32()
    st = lib().ref_capacity(C.byref(cfg), C.byref(params), workload.encode(), n, seed, slo_ms, C.byref(opts),
                            C.byref(qps), C.byref(mono), probes, cap, C.byref(npr))
    out = [(p.qps, bool(p.pass_), {f: getattr(p.report, f) for f, _ in _lib.Latency._fields_})
           for p in probes[:min(npr.value, cap)]]
    return st, qps.value, bool(mono.value), out
