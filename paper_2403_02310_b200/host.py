"""Python mirror of the reference simulator's host API over libss_host.so.

Names and argument meaning follow servesim (reference proj/include/servesim/*.hpp):
`ReplicaConfig`, `model_preset`, `make_trace`, `simulate`, `summarize`,
`iteration_time`, `compute_token_budget`, `get_next_chunk_size`,
`percentile`. Errors raise the reference's classes (ContractViolation,
OutOfKvBlocks, InfeasibleSlo). All logic runs in the C++ library; this module
only marshals arguments.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field, fields
from typing import Iterable, List, Optional, Sequence, Tuple

from . import _lib
from ._lib import CalibrationError, ContractViolation, InfeasibleSlo, OutOfKvBlocks, host_check, host_lib  # noqa: F401

POLICIES = {"request_level": 0, "vllm": 1, "orca": 2, "stall_free": 3}


@dataclass
class ReplicaConfig:
    """servesim::ReplicaConfig (reference core.hpp:105-125), same defaults."""

    scheduler: str = "stall_free"
    token_budget: int = 512
    max_batch_size: int = 512
    max_num_batched_tokens: int = 4096
    max_batch_size_orca: int = 0
    tp_degree: int = 1
    pp_degree: int = 1
    kv_blocks: int = 131072
    kv_block_size: int = 16
    tile_size: int = 256
    chunk_align: int = 32
    reserve_decode_tokens: int = 0
    kv_watermark_frac: float = 0.10
    pipeline_tbt_factor: float = 0.0
    hybrid_batching: bool = True

    def _c(self) -> _lib.ReplicaCfg:
        if self.scheduler not in POLICIES:
            raise ContractViolation(_lib.SS_INVALID_ARG, f"unknown scheduler {self.scheduler}")
        c = _lib.ReplicaCfg()
        for f in fields(self):
            v = getattr(self, f.name)
            if f.name == "scheduler":
                v = POLICIES[v]
            elif f.name == "hybrid_batching":
                v = int(bool(v))
            setattr(c, f.name, v)
        return c


@dataclass
class CostModelParams:
    """servesim::CostModelParams (reference costmodel.hpp:19-41)."""

    per_token_linear_ms: float = 0.0
    saturation_tokens: int = 1
    attn_prefill_quad_ms: float = 0.0
    attn_kv_read_ms: float = 0.0
    attn_decode_per_kv_ms: float = 0.0
    fixed_overhead_ms: float = 0.0
    tp_comm_ms: float = 0.0
    pp_send_ms: float = 0.0
    tile_size: int = 256
    tile_penalty_frac: float = 0.32

    def _c(self) -> _lib.CostParams:
        c = _lib.CostParams()
        for f in fields(self):
            setattr(c, f.name, getattr(self, f.name))
        return c


def model_preset(name: str) -> CostModelParams:
    """presets.cpp:8-66; plus "tiny", the unit-test clock of test_engine.cpp:14-25."""
    c = _lib.CostParams()
    host_check(host_lib().ssh_cost_preset(name.encode(), C.byref(c)))
    return CostModelParams(**{f.name: getattr(c, f.name) for f in fields(CostModelParams)})


@dataclass
class Request:
    arrival_us: int
    prompt_tokens: int
    output_tokens: int


@dataclass
class BatchEntry:
    """servesim::BatchEntry (core.hpp:73-78): kind 'decode' or 'prefill'."""

    request_id: int
    kind: str
    chunk_tokens: int
    prefix_tokens: int

    def _c(self) -> _lib.EntryRow:
        return _lib.EntryRow(self.request_id, 0 if self.kind == "decode" else 1, self.chunk_tokens, self.prefix_tokens)


def _rows(trace: Sequence[Request]):
    arr = (_lib.TraceRow * max(1, len(trace)))()
    for i, r in enumerate(trace):
        arr[i] = _lib.TraceRow(r.arrival_us, r.prompt_tokens, r.output_tokens)
    return arr


def make_trace(workload: str, qps: float, n: int, seed: int) -> List[Request]:
    """workload.cpp:73-84 with the presets of presets.cpp:82-100."""
    arr = (_lib.TraceRow * max(1, n))()
    host_check(host_lib().ssh_make_trace(workload.encode(), qps, n, seed, arr))
    return [Request(arr[i].arrival_us, arr[i].prompt_tokens, arr[i].output_tokens) for i in range(n)]


@dataclass
class Microbatch:
    entries: List[BatchEntry]
    iteration_ms: float
    issue_us: int

    @property
    def total_tokens(self) -> int:
        return sum(e.chunk_tokens for e in self.entries)


class SimReport:
    """Owns an ssh_report; event_log_jsonl() is byte-identical to the
    reference's SimReport::event_log_jsonl (engine.cpp:332-371)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)

    def __del__(self):
        try:
            if getattr(self, "_h", None) is not None and self._h.value:
                host_lib().ssh_report_free(self._h)
                self._h = None
        except Exception:  # interpreter shutdown
            pass

    def event_log_jsonl(self) -> str:
        n = C.c_size_t()
        p = host_lib().ssh_report_event_log(self._h, C.byref(n))
        return C.string_at(p, n.value).decode()

    def summarize(self, warmup_frac: float = 0.05) -> dict:
        out = _lib.Latency()
        host_check(host_lib().ssh_report_summary(self._h, warmup_frac, C.byref(out)))
        return out.as_dict()

    @property
    def num_microbatches(self) -> int:
        return host_lib().ssh_report_num_microbatches(self._h)

    @property
    def peak_blocks(self) -> int:
        return host_lib().ssh_report_peak_blocks(self._h)

    def microbatch(self, i: int) -> Microbatch:
        lib = host_lib()
        ms, issue = C.c_double(), C.c_int64()
        n = lib.ssh_report_microbatch(self._h, i, None, 0, C.byref(ms), C.byref(issue))
        if n < 0:
            raise IndexError(i)
        arr = (_lib.EntryRow * max(1, n))()
        lib.ssh_report_microbatch(self._h, i, arr, n, None, None)
        ents = [BatchEntry(a.request_id, "decode" if a.kind == 0 else "prefill", a.chunk_tokens, a.prefix_tokens)
                for a in arr[:n]]
        return Microbatch(ents, ms.value, issue.value)

    def microbatches(self) -> Iterable[Microbatch]:
        for i in range(self.num_microbatches):
            yield self.microbatch(i)


def _sim_opts(gpu, token_seed: int, keep_events: bool = False, check_block_tables: bool = False):
    """SimOpts for a cost-model clock (gpu None), one GPU context, or a pipeline group."""
    if gpu is not None and hasattr(gpu, "stages"):
        return _lib.SimOpts(int(keep_events), 0, None, token_seed, int(check_block_tables),
                            C.cast(gpu.handles, C.c_void_p), len(gpu.stages))
    h = gpu.handle.value if gpu is not None else None
    return _lib.SimOpts(int(keep_events), 0, h, token_seed, int(check_block_tables), None, 0)


def simulate(cfg: ReplicaConfig, params: CostModelParams, trace: Sequence[Request], *, keep_events: bool = True,
             gpu=None, token_seed: int = 0, check_block_tables: bool = False) -> SimReport:
    """engine.cpp:326-330. With gpu (a gpu.HybridForward) every issued batch runs
    the real forward and its measured time replaces iteration_time(); with a
    gpu.PipelineGroup (pp_degree stages) the batch runs through every stage and the
    slowest stage's time is the pipeline model's per-stage time."""
    opts = _sim_opts(gpu, token_seed, keep_events, check_block_tables)
    h = C.c_void_p()
    host_check(host_lib().ssh_simulate(C.byref(cfg._c()), C.byref(params._c()), _rows(trace), len(trace),
                                       C.byref(opts), C.byref(h)))
    return SimReport(h.value)


def iteration_time(entries: Sequence[BatchEntry], params: CostModelParams, tp: int = 1, pp: int = 1) -> float:
    arr = (_lib.EntryRow * max(1, len(entries)))(*[e._c() for e in entries])
    return host_lib().ssh_iteration_time(arr, len(entries), C.byref(params._c()), tp, pp)


def decode_reference_time(params: CostModelParams) -> float:
    return host_lib().ssh_decode_reference_time(C.byref(params._c()))


def compute_token_budget(t_max_ms: float, params: CostModelParams, pp_degree: int) -> int:
    out = C.c_int32()
    host_check(host_lib().ssh_compute_token_budget(t_max_ms, C.byref(params._c()), pp_degree, C.byref(out)))
    return out.value


@dataclass
class CalibrationResult:
    """servesim::CalibrationResult (costmodel.hpp:83-89)."""
    params: CostModelParams
    predicted_ms: List[float]
    relative_error: List[float]
    max_relative_error: float
    zeroed_terms: List[str]


CALIBRATION_TERMS = ["fixed_overhead_ms", "per_token_linear_ms", "attn_prefill_quad_ms", "attn_kv_read_ms",
                     "attn_decode_per_kv_ms"]


def _anchor_rows(anchors):
    keep = []
    rows = (_lib.AnchorRow * max(1, len(anchors)))()
    for i, (entries, ms) in enumerate(anchors):
        arr = (_lib.EntryRow * max(1, len(entries)))(*[e._c() for e in entries])
        keep.append(arr)
        rows[i].entries = C.cast(arr, C.POINTER(_lib.EntryRow))
        rows[i].n_entries = len(entries)
        rows[i].observed_ms = ms
    return rows, keep


def calibrate(anchors: Sequence[Tuple[Sequence[BatchEntry], float]], tile_size: int = 256,
              tile_penalty_frac: float = 0.32, max_saturation_tokens: int = 2048) -> CalibrationResult:
    """servesim::calibrate (calibrate.cpp:121-193): least-squares fit of the cost-model
    constants to (batch, observed ms) anchors — the measured B200 clock.
    Raises _lib.CalibrationError exactly where the reference throws CalibrationError."""
    rows, _keep = _anchor_rows(anchors)
    n = len(anchors)
    opts = _lib.CalibOpts(tile_size, tile_penalty_frac, max_saturation_tokens)
    out = _lib.CostParams()
    pred = (C.c_double * max(1, n))()
    rel = (C.c_double * max(1, n))()
    mx = C.c_double()
    mask = C.c_int32()
    host_check(host_lib().ssh_calibrate(rows, n, C.byref(opts), C.byref(out), pred, rel, C.byref(mx), C.byref(mask)))
    params = CostModelParams(**{f.name: getattr(out, f.name) for f in fields(CostModelParams)})
    return CalibrationResult(params, list(pred[:n]), list(rel[:n]), mx.value,
                             [t for i, t in enumerate(CALIBRATION_TERMS) if mask.value >> i & 1])


@dataclass
class CapacityProbe:
    qps: float
    passed: bool
    report: dict


@dataclass
class CapacityResult:
    """servesim::CapacityResult (metrics.hpp:57-61)."""
    qps: float
    monotone_warning: bool
    probes: List[CapacityProbe]


def slo_thresholds(params: CostModelParams) -> Tuple[float, float]:
    """metrics.cpp:60-63: (strict, relaxed) = (5x, 25x) the 32x4k decode iteration."""
    ref = decode_reference_time(params)
    return 5.0 * ref, 25.0 * ref


def capacity_search(cfg: ReplicaConfig, params: CostModelParams, workload: str, probe_requests: int, seed: int,
                    slo_ms: float, *, qps_low: float = 0.01, max_qps: float = 1024.0, rel_width: float = 0.05,
                    parallel: int = 1, gpu=None, token_seed: int = 0) -> CapacityResult:
    """servesim::capacity_search (metrics.cpp:70-138) with the CLI's probe (cli.cpp:434-439):
    make_trace(workload, qps, probe_requests, seed) -> simulate -> summarize -> meets_slo.
    params is the clock (a reference preset, or a calibrated B200 clock from clock.py);
    with gpu (a gpu.HybridForward) every probe runs real forwards. Raises InfeasibleSlo
    when qps_low fails."""
    opts = _lib.CapacityOpts(qps_low, max_qps, rel_width, parallel)
    sim = _sim_opts(gpu, token_seed)
    qps = C.c_double()
    mono = C.c_int32()
    cap = 256
    probes = (_lib.CapacityProbe * cap)()
    n = C.c_int32()
    host_check(host_lib().ssh_capacity_search(C.byref(cfg._c()), C.byref(params._c()), workload.encode(),
                                              probe_requests, seed, slo_ms, C.byref(opts), C.byref(sim),
                                              C.byref(qps), C.byref(mono), probes, cap, C.byref(n)))
    out = [CapacityProbe(p.qps, bool(p.pass_), {f: getattr(p.report, f) for f, _ in _lib.Latency._fields_})
           for p in probes[:min(n.value, cap)]]
    return CapacityResult(qps.value, bool(mono.value), out)


def get_next_chunk_size(prompt_tokens: int, prefill_done: int, token_budget: int, packed_tokens: int,
                        chunk_align: int) -> int:
    return host_lib().ssh_next_chunk_size(prompt_tokens, prefill_done, token_budget, packed_tokens, chunk_align)


def percentile(series: Sequence[float], p: float) -> float:
    arr = (C.c_double * max(1, len(series)))(*series)
    out = C.c_double()
    host_check(host_lib().ssh_percentile(arr, len(series), p, C.byref(out)))
    return out.value


class Descriptor:
    """Host-built ss_batch_desc (block tables, positions, slots, token ids)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)

    @classmethod
    def canonical(cls, tau: int, n_dec: int = 32, kv_each: int = 4096, chunk_prefix: int = 0, *,
                  block_size: int = 16, vocab: int, token_seed: int = 0) -> "Descriptor":
        h = C.c_void_p()
        host_check(host_lib().ssh_desc_canonical(tau, n_dec, kv_each, chunk_prefix, block_size, vocab, token_seed,
                                                 C.byref(h)))
        return cls(h.value)

    @classmethod
    def build(cls, entries: Sequence[BatchEntry], *, completes: Optional[Sequence[bool]] = None, block_size: int = 16,
              vocab: int, token_seed: int = 0) -> "Descriptor":
        arr = (_lib.EntryRow * max(1, len(entries)))(*[e._c() for e in entries])
        comp = None
        if completes is not None:
            comp = (C.c_int32 * max(1, len(entries)))(*[int(bool(x)) for x in completes])
        h = C.c_void_p()
        host_check(host_lib().ssh_desc_build(arr, len(entries), comp, block_size, vocab, token_seed, C.byref(h)))
        return cls(h.value)

    def __del__(self):
        try:
            if getattr(self, "_h", None) is not None and self._h.value:
                host_lib().ssh_desc_free(self._h)
                self._h = None
        except Exception:  # interpreter shutdown
            pass

    @property
    def view(self) -> _lib.BatchDesc:
        return host_lib().ssh_desc_view(self._h).contents

    @property
    def pool_blocks(self) -> int:
        return host_lib().ssh_desc_pool_blocks(self._h)

    def arrays(self) -> dict:
        """numpy copies of every descriptor array."""
        import numpy as np

        v = self.view
        E, T = v.num_entries, v.num_tokens
        a = lambda p, n, dt: np.ctypeslib.as_array(p, shape=(n,)).astype(dt).copy() if n > 0 else np.zeros(0, dt)
        return {
            "cu_q": a(v.cu_q, E + 1, np.int32), "ctx_len": a(v.ctx_len, E, np.int32), "pos": a(v.pos, T, np.int32),
            "token_ids": a(v.token_ids, T, np.int32), "slot": a(v.slot, T, np.int64),
            "block_table": a(v.block_table, E * v.max_blocks, np.int32).reshape(E, v.max_blocks),
            "out_rows": a(v.out_rows, v.n_out, np.int32),
        }


class Session:
    """Persistent ledger + block tables for replaying a micro-batch stream
    (ssh_session_*): entries keep their real request ids across steps."""

    def __init__(self, kv_blocks: int, *, block_size: int = 16, vocab: int, token_seed: int = 0):
        h = C.c_void_p()
        host_check(host_lib().ssh_session_create(kv_blocks, block_size, vocab, token_seed, C.byref(h)))
        self._h = h

    def step(self, entries: Sequence[BatchEntry], prompt_lens: Sequence[int]) -> Descriptor:
        arr = (_lib.EntryRow * len(entries))(*[e._c() for e in entries])
        pl = (C.c_int32 * len(entries))(*prompt_lens)
        h = C.c_void_p()
        host_check(host_lib().ssh_session_step(self._h, arr, len(entries), pl, C.byref(h)))
        return Descriptor(h.value)

    def release(self, request_id: int):
        host_check(host_lib().ssh_session_release(self._h, request_id))

    @property
    def peak_blocks(self) -> int:
        return host_lib().ssh_session_peak_blocks(self._h)

    def __del__(self):
        try:
            if getattr(self, "_h", None) is not None and self._h.value:
                host_lib().ssh_session_free(self._h)
                self._h = None
        except Exception:
            pass


def replay_plan(report: SimReport, trace: Sequence[Request]):
    """Yields (microbatch, prompt_lens, finished_ids) for executing a simulated
    stream in issue order: finished_ids are released after that step (pp = 1)."""
    for mb in report.microbatches():
        pl = [trace[e.request_id].prompt_tokens for e in mb.entries]
        done = []
        for e in mb.entries:
            r = trace[e.request_id]
            if e.kind == "prefill" and e.prefix_tokens + e.chunk_tokens == r.prompt_tokens and r.output_tokens == 1:
                done.append(e.request_id)
            elif e.kind == "decode" and e.prefix_tokens == r.prompt_tokens + r.output_tokens - 2:
                done.append(e.request_id)
        yield mb, pl, done
