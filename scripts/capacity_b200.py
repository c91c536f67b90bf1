"""Capacity under the strict TBT SLO with the B200 forward as the clock.

The paper's headline system metric: the highest request rate whose P99 TBT meets the SLO
(and whose median scheduling delay stays under 2 s), found by the reference's capacity search
(metrics.cpp:70-138, driven as cmd_capacity does at cli.cpp:421-460). Here every probe replays
make_trace(openchat, qps, n, seed) through the restated stall-free engine with the real
Mistral-7B-shaped forward on one B200 as the model step (GpuExecutor at the engine.cpp:227 seam),
so each probe's TBTs are measured device times.

SLO: strict = 5x the decode reference batch (32 decodes @ 4096, metrics.cpp:60-63), measured
on this B200. The same search on the reference's analytical A100 clock (its own SLO, 5x its own
decode reference) is printed beside it, with the same probe size and ladder start.

Probe size: the reference configs use 2048 requests per probe; with real forwards that is
~40k iterations per probe, so this run uses PROBE requests (default 256) for both clocks and
starts the ladder at QPS_LOW (default 1.0; below it every request runs alone, ~100k one-
sequence iterations per probe). Output: one JSON document on stdout.
  python scripts/capacity_b200.py > profiles/r02/capacity_mistral7b.json
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))

from paper_2403_02310_b200 import clock, gpu, host

MODEL = os.environ.get("MODEL", "mistral7b")
PROBE = int(os.environ.get("PROBE", "256"))
QPS_LOW = float(os.environ.get("QPS_LOW", "1.0"))
TAUS = [int(t) for t in os.environ.get("TAUS", "512").split(",")]
SEED = 42

shape = gpu.MODELS[MODEL]
params = host.model_preset(MODEL)
fwd = gpu.HybridForward(shape, weight_seed=1234)
dref = clock.time_batch(fwd, clock.decode_entries(32, 4096), reps=10)
slo_b200 = 5.0 * dref
slo_ref = host.slo_thresholds(params)[0]
per_block = shape.num_layers * 2 * shape.num_kv_heads * 16 * shape.head_dim * 2
pool = int(min(40000, 90e9 // per_block))
fwd.kv_alloc(pool)

out = {
    "model": f"{MODEL}-shaped random-init, TP1, one B200",
    "workload": f"openchat (make_trace, seed {SEED}), {PROBE} requests per probe",
    "search": {"qps_low": QPS_LOW, "max_qps": 1024.0, "rel_width": 0.05, "parallel": 1,
               "slo_rule": "P99 TBT <= slo and median scheduling delay <= 2 s (metrics.cpp meets_slo)"},
    "decode_reference_ms": {"b200_measured": dref, "reference_a100_clock": host.decode_reference_time(params)},
    "strict_slo_ms": {"b200": slo_b200, "reference_a100_clock": slo_ref},
    "kv_blocks": pool,
    "runs": [],
}
for tau in TAUS:
    cfg = host.ReplicaConfig(token_budget=tau, kv_blocks=pool)
    t0 = time.time()
    try:
        r = host.capacity_search(cfg, params, "openchat", PROBE, SEED, slo_b200, qps_low=QPS_LOW, gpu=fwd,
                                 token_seed=SEED)
        b200 = {"capacity_qps": r.qps, "monotone_warning": r.monotone_warning,
                "probes": [{"qps": p.qps, "pass": p.passed,
                            "tbt_p99_ms": p.report.get("tbt_p99_ms"), "sched_delay_median_ms":
                                p.report.get("sched_delay_median_ms"), "throughput_tps": p.report.get("throughput_tps")}
                           for p in r.probes]}
    except host.InfeasibleSlo as e:
        b200 = {"capacity_qps": 0.0, "infeasible": str(e)}
    b200["wall_s"] = time.time() - t0
    ref = host.capacity_search(cfg, params, "openchat", PROBE, SEED, slo_ref, qps_low=QPS_LOW, parallel=8)
    # the B200 forward against the reference's (A100) SLO too: same absolute bar
    out["runs"].append({"token_budget": tau, "b200_forward_clock": b200,
                        "reference_a100_clock": {"capacity_qps": ref.qps, "probes": [p.qps for p in ref.probes]}})
    print(f"tau={tau}: B200 {b200.get('capacity_qps')} qps (slo {slo_b200:.2f} ms), reference clock {ref.qps} qps "
          f"(slo {slo_ref:.1f} ms), {b200['wall_s']:.0f} s", file=sys.stderr, flush=True)
fwd.close()
print(json.dumps(out, indent=1))
