#!/usr/bin/env python
"""Benchmark of the B200 hybrid-batch forward (Sarathi-Serve stall-free iteration).

Workload (BASELINE.json configs[1]): Mistral-7B-shaped random-init model, token
budget tau = 512, the reference's canonical hybrid batch (reference
proj/src/sched.cpp:159-169): 32 decodes at a 4096-token context plus one
prompt-completing chunk of tau - 32 = 480 tokens at prefix 0. One step = one
forward of that batch through all 32 layers + LM head on the 33 logit rows.
Tensor-parallel over N GPUs (one process per GPU). The TP all-reduce runs inside
the library on one of two transports: the CUDA-IPC peer-memory collective fused
with the residual add (default, --tp-comm ipc) or NCCL all-reduce + a residual-add
kernel (--tp-comm nccl). value = batch tokens / max-over-ranks step time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the fp32 CPU forward (oracle/, the CPU restatement of
the path; the reference simulator itself has no numeric forward) on the host
cores: every step is one full forward of the same batch (all L layers + LM head).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
METRIC = "hybrid-batch tokens/s & iter latency @budget 512/2048, 1-8 B200; P99 TBT"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return dict(PEAKS_FALLBACK), "fallback"


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, device: int):
        self.device, self.samples, self.proc, self.t = device, [], None, None

    def start(self):
        cmd = ["nvidia-smi", "-i", str(self.device),
               "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
               "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
               "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
               "--format=csv,noheader,nounits", "-lms", "50"]
        try:
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                self.samples.append((time.time(), parts))

    def stop(self, t0, t1):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        self.t.join(timeout=2)
        win = [p for (t, p) in self.samples if t0 <= t <= t1] or [p for (_, p) in self.samples]
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = sorted(v for v in (num(p[0]) for p in win) if v is not None)
        smax = max((v for v in (num(p[1]) for p in win) if v is not None), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for p in win for i in range(4) if p[4 + i].lower() in ("active", "1", "yes")})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": smax, "reasons": reasons,
                "samples": len(win)}


def algorithmic_work(shape, desc_arrays, tp):
    """SURVEY 8(d) per-GPU algorithmic bytes / flops of one canonical-batch step."""
    L, h, hd = shape.num_layers, shape.hidden, shape.head_dim
    nq, nkv = shape.num_q_heads // tp, shape.num_kv_heads // tp
    T = len(desc_arrays["pos"])
    n_out = len(desc_arrays["out_rows"])
    ctx = desc_arrays["ctx_len"].astype(float)
    ntok = (desc_arrays["cu_q"][1:] - desc_arrays["cu_q"][:-1]).astype(float)
    cached = float((ctx - ntok).sum())
    p_layer = shape.params_per_layer() / tp
    kv_tok = 2 * nkv * hd * 2  # K+V bytes per token per layer
    bytes_w = 2 * (L * p_layer + shape.vocab * h / tp)
    bytes_kv_read = L * kv_tok * cached
    bytes_kv_write = L * kv_tok * T
    # visible (query, key) pairs: token at position p sees p + 1 keys
    pairs = float((desc_arrays["pos"].astype(float) + 1).sum())
    flops = 2 * T * L * p_layer + 2 * n_out * shape.vocab * h / tp + 4 * hd * nq * L * pairs
    per_layer = {
        "gemm_qkv": 2.0 * T * h * (nq + 2 * nkv) * hd, "gemm_o": 2.0 * T * nq * hd * h,
        "gemm_gate_up": 2.0 * T * h * 2 * shape.ffn / tp, "gemm_down": 2.0 * T * shape.ffn / tp * h,
        "attention_bytes": kv_tok * (cached + T) + 2 * 2 * T * nq * hd,
        "attention_flops": 4 * hd * nq * pairs,
        "lm_head": 2.0 * n_out * shape.vocab / tp * h,
    }
    # the fused projection chain (one launch per layer at TP = 1): O + gate/up + down of the
    # layer and the next layer's QKV (the last layer's chain has no QKV); per step
    per_layer["gemm_chain_step"] = (L * (per_layer["gemm_o"] + per_layer["gemm_gate_up"] + per_layer["gemm_down"])
                                    + (L - 1) * per_layer["gemm_qkv"])
    return {"bytes": bytes_w + bytes_kv_read + bytes_kv_write, "flops": flops, "per_layer": per_layer,
            "T": T, "n_out": n_out}


def run_ours(args):
    import numpy as np
    import torch

    from paper_2403_02310_b200 import gpu, host

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}; launch N>1 under torch.distributed.run")
    if os.environ.get("SS_BENCH_ONE_DEVICE"):  # dev: every rank on cuda:0 (checks the N>1 path on one GPU)
        local = 0
    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("gloo", init_method="env://")
        pg = dist
    shape = gpu.MODELS[args.model]
    if args.layers:
        shape = shape.with_layers(args.layers)
    nccl_id = None
    if world > 1 and args.tp_comm == "nccl":
        buf = [gpu.nccl_unique_id() if rank == 0 else None]
        pg.broadcast_object_list(buf, src=0)
        nccl_id = buf[0]
    fwd = gpu.HybridForward(shape, tp_rank=rank, tp_size=world, nccl_id=nccl_id, weight_seed=1234, device=local)
    if world > 1 and args.tp_comm == "ipc":
        def allgather(b):
            out = [None] * world
            pg.all_gather_object(out, b)
            return out

        fwd.ipc_connect(allgather, max_tokens=max(8192, args.tau))
    desc = host.Descriptor.canonical(args.tau, 32, 4096, args.chunk_prefix, vocab=shape.vocab, token_seed=7)
    arrays = desc.arrays()
    fwd.kv_alloc(desc.pool_blocks)
    fwd.fill_descriptor_prefixes(desc, seed=5)
    batch = fwd.upload(desc)
    st = fwd.torch_stream()
    work = algorithmic_work(shape, arrays, world)

    def barrier():
        fwd.synchronize()
        if pg:
            pg.barrier()

    def max_over_ranks(v):
        if not pg:
            return v
        t = torch.tensor([v], dtype=torch.float64)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        fwd.enqueue(batch)
    if args.profile_step:
        # one steady-state step bracketed by cudaProfilerStart/Stop, for
        # `ncu --profile-from-start off` launch lists and captures
        fwd.synchronize()
        torch.cuda.profiler.start()
        fwd.enqueue(batch)
        fwd.synchronize()
        torch.cuda.profiler.stop()
        batch.free()
        fwd.close()
        return
    clock = ClockSampler(local)
    clock.start()
    time.sleep(0.2)
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0 = fwd.launch_count
    t_wall0 = time.time()
    e0.record(st)
    for _ in range(args.steps):
        fwd.enqueue(batch)
    e1.record(st)
    barrier()
    torch.cuda.synchronize()
    t_wall1 = time.time()
    launches = fwd.launch_count - n0
    ms_step = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    clocks = clock.stop(t_wall0, t_wall1)
    _, toks = fwd.read_outputs(batch)
    assert np.all((toks >= 0) & (toks < shape.vocab))

    # per-kernel-class device time: a second pass over the same K steps with CUDA
    # events around every launch on the library stream
    fwd.set_profiling(True)
    fwd.kernel_times(reset=True)
    barrier()
    for _ in range(args.steps):
        fwd.enqueue(batch)
    barrier()
    kt = fwd.kernel_times(reset=True)
    fwd.set_profiling(False)
    prof_total = sum(v[0] for v in kt.values())

    # end to end through the public C ABI: host descriptor in, next tokens out
    view = desc.view
    h2d = sum(a.nbytes for k, a in arrays.items())
    d2h = 4 * work["n_out"]
    def e2e_time():
        for _ in range(3):  # the shape's graph is captured on its second forward
            fwd.forward(desc, logits=False)
        barrier()
        call_ms = []
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            call_ms.append(fwd.forward(view, logits=False)[2])  # the call's own device time (its events)
        barrier()
        wall = max_over_ranks((time.perf_counter() - t0) * 1e3 / args.e2e_steps)
        return wall, max_over_ranks(sum(call_ms) / len(call_ms))

    e2e_ms, e2e_call_dev = e2e_time()  # CUDA graph replays (default)
    fwd.set_graphs(False)
    e2e_eager_ms, e2e_eager_dev = e2e_time()  # the same calls with eager launches, for the graph effect
    fwd.set_graphs(True)

    peaks, peak_src = load_peaks()
    T = work["T"]
    L = shape.num_layers
    kernels = {}
    for k, (ms, n) in kt.items():
        if n == 0:
            continue
        ent = {"ms_per_step": ms / args.steps, "launches_per_step": n / args.steps, "share": ms / prof_total}
        pl = work["per_layer"]
        # per-layer classes: time per layer (attention is one or two kernel launches per layer)
        per_layer_cls = k in ("gemm_qkv", "gemm_o", "gemm_gate_up", "gemm_down", "attention")
        avg = ms / args.steps / L if per_layer_cls else ms / n
        if k in ("gemm_qkv", "gemm_o", "gemm_gate_up", "gemm_down", "lm_head"):
            ent["tflops"] = pl[k] / (avg * 1e-3) / 1e12
        if k == "gemm_chain":  # flops of every chain launch of the step over their total time
            ent["tflops"] = pl["gemm_chain_step"] / (ms / args.steps * 1e-3) / 1e12
            ent["flops_per_launch"] = pl["gemm_chain_step"] / max(1.0, n / args.steps)
        if k == "attention":
            ent["gbs"] = pl["attention_bytes"] / (avg * 1e-3) / 1e9
        kernels[k] = ent
    # dominant compute kernel (the TP collective class has no roofline of its own here)
    dom = max((k for k in kernels if "tflops" in kernels[k] or "gbs" in kernels[k]), key=lambda k: kernels[k]["share"])
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):
        with open(tfile) as f:
            traffic = json.load(f).get(args.model, {}).get(dom)
    # Peak basis: the burst figures (cuBLAS alone, ~max clock) when the timed region ran at
    # >= 95% of the max SM clock, else the sustained (power-capped) figure; both reported.
    burst_clock = bool(clocks.get("sm_mhz") and clocks.get("sm_max_mhz")
                       and clocks["sm_mhz"] >= 0.95 * clocks["sm_max_mhz"])
    if dom == "attention":
        roof = {"bound": "hbm", "achieved": kernels[dom]["gbs"], "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "peak_basis": "measured copy bandwidth"}
    else:
        ach = kernels[dom]["tflops"]
        peak = peaks["bf16_tflops"] if burst_clock else peaks["bf16_tflops_sustained"]
        roof = {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                "peak_basis": ("burst (timed region at >= 95% of max SM clock)" if burst_clock
                               else "sustained (timed region below 95% of max SM clock)"),
                "frac_of_burst": ach / peaks["bf16_tflops"],
                "frac_of_sustained": ach / peaks["bf16_tflops_sustained"]}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["traffic"] = traffic
    roof["kernel"] = dom
    roof["peak_source"] = peak_src
    whole_roof_ms = max(work["bytes"] / (peaks["hbm_gbs"] * 1e9), work["flops"] / (peaks["bf16_tflops"] * 1e12)) * 1e3

    # the metric's other operating points, same timing (BASELINE: budgets 512 and 2048;
    # the chunk-at-cached-prefix variant of SURVEY 8(d))
    extra = {}
    if not args.no_extra_configs:
        for tau_x, pre_x in ((2048, 0), (args.tau, 2048)):
            if (tau_x, pre_x) != (args.tau, args.chunk_prefix):
                extra[f"tau{tau_x}_prefix{pre_x}"] = time_canonical(
                    fwd, shape, tau_x, pre_x, min(args.steps, 10), 3, peaks, world, barrier, max_over_ranks)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(shape, args.tau, args.chunk_prefix, budget_s=args.cpu_budget_s)

    tbt = None
    if world == 1 and args.tbt_requests > 0:
        batch.free()
        tbt = closed_loop_tbt(fwd, args.model, args.tau, args.tbt_requests, args.tbt_qps)
        # the same closed loop with eager launches (graphs off): P99 TBT / wall beside it
        fwd.set_graphs(False)
        t_eager = closed_loop_tbt(fwd, args.model, args.tau, args.tbt_requests, args.tbt_qps, cost_clock=False)
        fwd.set_graphs(True)
        tbt["graphs_off"] = {k: t_eager[k] for k in ("p99_ms", "median_ms", "iter_ms_median", "wall_s")}
        tbt["graphs"] = dict(zip(("captures", "replays"), fwd.graph_stats()))

    out = {
        "metric": METRIC, "value": T / (ms_step * 1e-3), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (counter-based random-init weights, synthetic 4k-token caches, hashed token ids)",
        "config": {"workload": f"canonical hybrid batch: 32 decodes @4096 ctx + 1 chunk of {args.tau - 32} tokens "
                               f"@prefix {args.chunk_prefix} (reference sched.cpp:159-169)",
                   "model": f"{args.model}-shaped (L={L}, h={shape.hidden}, q={shape.num_q_heads}, "
                            f"kv={shape.num_kv_heads}, hd={shape.head_dim}, ffn={shape.ffn}, V={shape.vocab})",
                   "token_budget": args.tau, "tokens_per_step": T, "logit_rows": work["n_out"],
                   "parallelism": f"tp{world}" + (f" ({args.tp_comm} all-reduce)" if world > 1 else ""),
                   "l2": "inputs larger than L2 (all weights + KV re-read every step)",
                   "gpu_launches_per_step": launches / args.steps},
        "e2e": {"value": T / (e2e_ms * 1e-3), "unit": "tokens/s", "ms_per_step": e2e_ms, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "api": "ss_forward_hybrid (host descriptor arrays -> next tokens)",
                "graphs": "CUDA graph replay of the batch shape (ss_set_graphs, default on)",
                "gap_vs_device_ms": e2e_ms - ms_step,
                # host time per call: wall minus the call's own device time (H2D .. D2H events);
                # the gap above also counts that back-to-back device steps overlap (PDL)
                "call_device_ms": e2e_call_dev, "gap_vs_call_device_ms": e2e_ms - e2e_call_dev,
                "graphs_off": {"value": T / (e2e_eager_ms * 1e-3), "ms_per_step": e2e_eager_ms,
                               "gap_vs_device_ms": e2e_eager_ms - ms_step,
                               "gap_vs_call_device_ms": e2e_eager_ms - e2e_eager_dev}},
        "gpu_launches": launches,
        "roofline": roof,
        "whole_step_roofline": {"ms": whole_roof_ms, "frac": whole_roof_ms / ms_step, "alg_bytes": work["bytes"],
                                "alg_flops": work["flops"]},
        "kernels": kernels,
        "other_operating_points": extra,
        "clocks": clocks,
        "cpu_baseline": cpu,
        "cost_model_ms": reference_cost_model_ms(args.model, args.tau, args.chunk_prefix, world),
        "tbt": tbt,
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    if tbt is None:
        batch.free()
    fwd.close()
    if pg:
        pg.destroy_process_group()


def time_canonical(fwd, shape, tau, prefix, steps, warmup, peaks, world, sync, max_over_ranks):
    """Device time of another canonical batch (the metric's second budget, or the chunk
    at a cached prefix, sched.cpp:159-169 / PAPER.md:532) with the same event timing."""
    import torch

    from paper_2403_02310_b200 import host

    desc = host.Descriptor.canonical(tau, 32, 4096, prefix, vocab=shape.vocab, token_seed=7)
    fwd.kv_alloc(desc.pool_blocks)
    fwd.fill_descriptor_prefixes(desc, seed=5)
    b = fwd.upload(desc)
    st = fwd.torch_stream()
    for _ in range(warmup):
        fwd.enqueue(b)
    sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        fwd.enqueue(b)
    e1.record(st)
    sync()
    ms = max_over_ranks(e0.elapsed_time(e1) / steps)
    work = algorithmic_work(shape, desc.arrays(), world)
    roof = max(work["bytes"] / (peaks["hbm_gbs"] * 1e9), work["flops"] / (peaks["bf16_tflops"] * 1e12)) * 1e3
    b.free()
    return {"workload": f"32 decodes @4096 + chunk of {tau - 32} @prefix {prefix}", "token_budget": tau,
            "ms_per_step": ms, "value": tau / (ms * 1e-3), "unit": "tokens/s", "steps": steps,
            "whole_step_roofline": {"ms": roof, "frac": roof / ms}}


def closed_loop_tbt(fwd, model, tau, n_requests, qps, seed=42, cost_clock=True):
    """P99 TBT from a replayed synthetic trace: the restated engine (byte-identical
    to the reference's, tests/test_host_parity.py) runs the stall-free schedule
    with the real B200 forward as its model step (engine.cpp:227 seam); every
    iteration's measured device time drives the clock. summarize() follows
    metrics.cpp:23-59 (nearest-rank P99, 5% warm-up). The same trace under the
    reference's analytical clock is reported beside it."""
    from paper_2403_02310_b200 import host

    trace = host.make_trace("openchat", qps, n_requests, seed)
    params = host.model_preset(model if model != "tiny" else "tiny")
    shape = fwd.shape
    per_block = shape.num_layers * 2 * (shape.num_kv_heads // fwd.tp_size) * 16 * shape.head_dim * 2
    pool = 65536 if model == "tiny" else int(min(40000, 90e9 // per_block))  # <= 90 GB of KV pool
    fwd.kv_alloc(pool)
    cfg = host.ReplicaConfig(token_budget=tau, kv_blocks=pool)
    t0 = time.perf_counter()
    rep = host.simulate(cfg, params, trace, gpu=fwd, token_seed=seed, keep_events=False)
    wall = time.perf_counter() - t0
    s = rep.summarize()
    iters = [mb.iteration_ms for mb in rep.microbatches()]
    out = {"p99_ms": s["tbt_p99_ms"], "median_ms": s["tbt_median_ms"], "ttft_median_ms": s["ttft_median_ms"],
            "throughput_tps": s["throughput_tps"], "iterations": len(iters),
            "iter_ms_median": sorted(iters)[len(iters) // 2], "iter_ms_max": max(iters), "wall_s": wall,
            "trace": f"openchat (median prompt 1730 / P90 5696, output 415 / 834), n={n_requests}, qps={qps}, "
                     f"seed={seed}, stall_free tau={tau}"}
    if cost_clock:
        ref = host.simulate(cfg, params, trace, keep_events=False).summarize()
        out["cost_model_clock"] = {"p99_ms": ref["tbt_p99_ms"], "ttft_median_ms": ref["ttft_median_ms"],
                                   "throughput_tps": ref["throughput_tps"]}
    return out


def reference_cost_model_ms(model, tau, chunk_prefix, tp):
    """The reference's own iteration_time() for the same batch (A100-calibrated synthetic)."""
    from paper_2403_02310_b200 import host

    try:
        ents = [host.BatchEntry(i, "decode", 1, 4096) for i in range(32)] + [
            host.BatchEntry(32, "prefill", tau - 32, chunk_prefix)]
        return host.iteration_time(ents, host.model_preset(model), tp)
    except Exception:
        return None


def cpu_baseline(shape, tau, chunk_prefix, budget_s=20.0, steps=None, warmup=1):
    """fp32 oracle forward on the host cores: one decoder layer of the canonical
    batch per sample, extrapolated x L (the full model does not fit a bounded run)."""
    from oracle.forward import Oracle, threads
    from paper_2403_02310_b200 import host

    desc = host.Descriptor.canonical(tau, 32, 4096, chunk_prefix, vocab=shape.vocab, token_seed=7)
    orc = Oracle(shape, weight_seed=1234, num_blocks=desc.pool_blocks, layers=1, with_head=False)
    orc.fill_descriptor_prefixes(desc, seed=5)
    for _ in range(warmup):
        orc.forward(desc)
    times = []
    t_start = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        orc.forward(desc)
        times.append(time.perf_counter() - t0)
        if steps is not None and len(times) >= steps:
            break
        if steps is None and time.perf_counter() - t_start > budget_s * 0.5 and len(times) >= 2:
            break
    orc.close()
    per_layer = sum(times) / len(times)
    T = tau
    return {"value": T / (per_layer * shape.num_layers), "unit": "tokens/s", "cores": threads(), "kind": "port",
            "cpu": cpu_model(),
            "sample": f"fp32 oracle, 1 of {shape.num_layers} decoder layers of the canonical tau={tau} batch "
                      f"({len(times)} reps, {per_layer:.3f} s/layer), extrapolated x{shape.num_layers}; LM head omitted",
            "s_per_layer": per_layer}


def cpu_model():
    """CPU model string and logical core count of this host (for the CPU legs)."""
    name = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.lower().startswith("model name"):
                    name = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"model": name, "logical_cpus": os.cpu_count()}


def run_reference(args):
    """The reference arm: the path's CPU implementation (the fp32 oracle, oracle/ — the
    reference simulator itself has no numeric forward) on the host cores, every step one
    FULL forward of the same canonical batch: all L decoder layers + the LM head, no
    extrapolation. Loads no product library: the descriptor comes from
    oracle/canonical.py, the shape table is plain data."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle.canonical import CanonicalDesc
    from oracle.forward import Oracle, threads
    from paper_2403_02310_b200.gpu import MODELS  # shape table only (no library is loaded)

    shape = MODELS[args.model]
    desc = CanonicalDesc(args.tau, 32, 4096, args.chunk_prefix, vocab=shape.vocab, token_seed=7)
    orc = Oracle(shape, weight_seed=1234, num_blocks=desc.pool_blocks)
    orc.fill_descriptor_prefixes(desc, seed=5)
    # CPU warm-up: one forward pages in weights and KV; more would only lengthen the run
    warm = min(args.warmup, 1)
    for _ in range(warm):
        orc.forward(desc)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        lg = orc.forward(desc)
        times.append(time.perf_counter() - t0)
    orc.close()
    assert lg.shape == (33, shape.vocab)
    ms_step = sum(times) / len(times) * 1e3
    value = args.tau / (ms_step * 1e-3)
    cpu = cpu_model()
    out = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": warm, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"canonical hybrid batch: 32 decodes @4096 ctx + 1 chunk of {args.tau - 32} tokens "
                               f"@prefix {args.chunk_prefix} (same as --impl ours)",
                   "model": f"{args.model}-shaped", "token_budget": args.tau, "tokens_per_step": args.tau,
                   "parallelism": "host cores (OpenMP)"},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads(), "kind": "port",
                         "cpu": cpu,
                         "sample": f"every step = one full forward of the canonical batch on the fp32 oracle "
                                   f"(all {shape.num_layers} decoder layers + LM head on the 33 logit rows, no "
                                   f"extrapolation; the reference simulator has no numeric forward); "
                                   f"{warm} untimed warm-up step(s)"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--model", default="mistral7b")
    ap.add_argument("--tau", type=int, default=512)
    ap.add_argument("--chunk-prefix", type=int, default=0)
    ap.add_argument("--layers", type=int, default=0, help="debug only: truncate depth (invalidates the metric)")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--cpu-budget-s", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra-configs", action="store_true", help="skip the tau=2048 / chunk@2048 lines")
    ap.add_argument("--tbt-requests", type=int, default=48, help="closed-loop P99 TBT trace size (0: skip)")
    ap.add_argument("--tbt-qps", type=float, default=4.0)
    ap.add_argument("--tp-comm", choices=["ipc", "nccl"], default="ipc",
                    help="tp > 1 transport: CUDA-IPC peer-memory all-reduce fused with the residual add (default) "
                         "or NCCL all-reduce + residual-add kernel")
    ap.add_argument("--profile-step", action="store_true",
                    help="profiling only: after warm-up run one step between cudaProfilerStart/Stop and exit")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
