"""The measured B200 clock: one-time profiling -> calibrated cost model -> token budget.

Sarathi-Serve picks its token budget tau from one-time profiling of the model step
(PAPER.md:535): the largest tau whose hybrid-batch iteration meets the TBT SLO.
The reference does this on its analytical A100 constants: compute_token_budget
(sched.cpp:154-175) over iteration_time with a preset, SLOs from
slo_thresholds (metrics.cpp:60-63: strict 5x / relaxed 25x the 32x4k decode
batch). Here the same pipeline runs on the real B200 forward:

  1. time anchor batches (decode-only, prefill-only, chunk-with-prefix,
     canonical hybrids) through ss_forward_hybrid's device path;
  2. fit the reference's five constants with calibrate (calibrate.cpp:121-193,
     host.calibrate);
  3. derive the SLOs from the measured decode reference batch and pick tau
     with compute_token_budget on the calibrated constants, and, directly, by
     searching the measured canonical batch time.
"""
from __future__ import annotations

import statistics
from typing import Dict, List, Sequence, Tuple

from . import host


def decode_entries(count: int, kv: int) -> List[host.BatchEntry]:
    return [host.BatchEntry(i, "decode", 1, kv) for i in range(count)]


def chunk_entries(tokens: int, prefix: int = 0) -> List[host.BatchEntry]:
    return [host.BatchEntry(0, "prefill", tokens, prefix)]


def canonical_entries(tau: int, n_dec: int = 32, kv: int = 4096, chunk_prefix: int = 0) -> List[host.BatchEntry]:
    """sched.cpp:159-169: n_dec decodes at kv plus one chunk of tau - n_dec tokens."""
    return decode_entries(n_dec, kv) + [host.BatchEntry(n_dec, "prefill", tau - n_dec, chunk_prefix)]


def default_anchors() -> List[Tuple[str, List[host.BatchEntry]]]:
    """Both regimes and every term of the model: memory-bound decodes, compute-bound
    prefills (incl. one below saturation), a chunk re-reading its prefix, hybrids."""
    a = [(f"decode {b}x4096", decode_entries(b, 4096)) for b in (1, 8, 32)]
    a += [(f"decode 32x{kv}", decode_entries(32, kv)) for kv in (1024, 2048)]
    a += [(f"prefill {n}", chunk_entries(n)) for n in (128, 256, 512, 1024, 2048, 4096)]
    a += [(f"chunk 512@{p}", chunk_entries(512, p)) for p in (2048, 4096)]
    a += [(f"hybrid tau={t}", canonical_entries(t)) for t in (256, 512, 1024, 2048)]
    return a


def time_batch(fwd, entries: Sequence[host.BatchEntry], reps: int = 8, warmup: int = 2, seed: int = 5) -> float:
    """Median device ms of the forward of one batch (inputs resident, CUDA events on
    the library stream). The pool must already hold desc.pool_blocks blocks."""
    import torch

    d = host.Descriptor.build(entries, vocab=fwd.shape.vocab, token_seed=seed)
    if d.pool_blocks > fwd.kv_blocks:
        fwd.kv_alloc(d.pool_blocks)
    fwd.fill_descriptor_prefixes(d, seed=seed)
    b = fwd.upload(d)
    st = fwd.torch_stream()
    for _ in range(warmup):
        fwd.enqueue(b)
    fwd.synchronize()
    times = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fwd.enqueue(b)
        e1.record(st)
        fwd.synchronize()
        times.append(e0.elapsed_time(e1))
    b.free()
    return statistics.median(times)


def measured_budget(fwd, t_max_ms: float, hi: int = 8192, step: int = 32, **kw) -> Tuple[int, float]:
    """Largest tau (multiple of `step`, >= 64) whose MEASURED canonical batch meets t_max
    (binary search; the canonical time is monotone in tau up to noise)."""
    lo_ok, lo_ms = 0, 0.0
    lo, top = 64 // step, hi // step
    while lo <= top:
        mid = (lo + top) // 2
        ms = time_batch(fwd, canonical_entries(mid * step), **kw)
        if ms <= t_max_ms:
            lo_ok, lo_ms = mid * step, ms
            lo = mid + 1
        else:
            top = mid - 1
    return lo_ok, lo_ms


def b200_clock(fwd, anchors=None, reps: int = 8) -> Dict:
    anchors = anchors or default_anchors()
    rows = []
    for name, ents in anchors:
        rows.append((name, ents, time_batch(fwd, ents, reps=reps)))
    cal = host.calibrate([(e, ms) for _, e, ms in rows])
    p = cal.params
    dref_measured = time_batch(fwd, decode_entries(32, 4096), reps=reps)
    out = {
        "anchors": [{"name": n, "tokens": sum(e.chunk_tokens for e in es), "measured_ms": ms,
                     "calibrated_ms": pr, "rel_err": re}
                    for (n, es, ms), pr, re in zip(rows, cal.predicted_ms, cal.relative_error)],
        "calibrated": {f: getattr(p, f) for f in ("fixed_overhead_ms", "per_token_linear_ms", "saturation_tokens",
                                                  "attn_prefill_quad_ms", "attn_kv_read_ms",
                                                  "attn_decode_per_kv_ms", "tile_size", "tile_penalty_frac")},
        "zeroed_terms": cal.zeroed_terms,
        "max_relative_error": cal.max_relative_error,
        "decode_reference_ms": {"measured": dref_measured, "calibrated": host.decode_reference_time(p)},
        "slo": {},
    }
    for label, mult in (("strict", 5.0), ("relaxed", 25.0)):  # metrics.cpp:60-63
        t_max = mult * dref_measured
        try:
            tau_model = host.compute_token_budget(t_max, p, 1)
        except host.InfeasibleSlo:
            tau_model = None
        tau_meas, ms = measured_budget(fwd, t_max, reps=max(3, reps // 2))
        out["slo"][label] = {"t_max_ms": t_max, "tau_calibrated_model": tau_model, "tau_measured": tau_meas,
                             "measured_ms_at_tau": ms}
    return out


def tile_curve(fwd, tokens: Sequence[int], reps: int = 6) -> List[Tuple[int, float]]:
    """Prefill-only forward time vs T around tile boundaries (the reference's tile
    penalty, tile 256 + 32%: what tcgen05 256-row pair tiles cost)."""
    return [(t, time_batch(fwd, chunk_entries(t), reps=reps)) for t in tokens]
