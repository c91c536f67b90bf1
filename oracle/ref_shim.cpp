// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the reference simulator (servesim) compiled from its
// own sources under /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libservesim_ref.so. It exposes the reference's host path with
// the same plain-C argument structs as include/ss_host.h so the parity tests
// can drive both implementations through identical inputs:
//   ref_simulate        -> servesim::simulate + SimReport::event_log_jsonl
//                          (reference engine.cpp:326-371)
//   ref_summary         -> servesim::summarize (metrics.cpp:23-59)
//   ref_make_trace      -> servesim::make_trace (workload.cpp:73-84)
//   ref_iteration_time  -> servesim::iteration_time (costmodel.cpp:39-56)
//   ref_token_budget    -> servesim::compute_token_budget (sched.cpp:154-175)
//   ref_cost_preset     -> servesim::model_preset (presets.cpp:71-77)
//   ref_calibrate       -> servesim::calibrate (calibrate.cpp:121-193)
//   ref_capacity        -> servesim::capacity_search with the CLI's probe
//                          (metrics.cpp:70-138, cli.cpp:434-439)
#include <cstring>
#include <string>

#include "servesim/costmodel.hpp"
#include "servesim/engine.hpp"
#include "servesim/metrics.hpp"
#include "servesim/presets.hpp"
#include "servesim/sched.hpp"
#include "servesim/workload.hpp"
#include "../include/ss_host.h"

using namespace servesim;

namespace {

thread_local std::string g_err;

ReplicaConfig to_cfg(const ssh_replica_cfg& c) {
    ReplicaConfig r;
    r.scheduler = static_cast<SchedulerPolicy>(c.scheduler);
    r.token_budget = c.token_budget;
    r.max_batch_size = c.max_batch_size;
    r.max_num_batched_tokens = c.max_num_batched_tokens;
    r.max_batch_size_orca = c.max_batch_size_orca;
    r.tp_degree = c.tp_degree;
    r.pp_degree = c.pp_degree;
    r.kv_blocks = c.kv_blocks;
    r.kv_block_size = c.kv_block_size;
    r.tile_size = c.tile_size;
    r.chunk_align = c.chunk_align;
    r.reserve_decode_tokens = c.reserve_decode_tokens;
    r.kv_watermark_frac = c.kv_watermark_frac;
    r.pipeline_tbt_factor = c.pipeline_tbt_factor;
    r.hybrid_batching = c.hybrid_batching != 0;
    return r;
}

CostModelParams to_params(const ssh_cost_params& c) {
    CostModelParams p;
    p.per_token_linear_ms = c.per_token_linear_ms;
    p.saturation_tokens = c.saturation_tokens;
    p.attn_prefill_quad_ms = c.attn_prefill_quad_ms;
    p.attn_kv_read_ms = c.attn_kv_read_ms;
    p.attn_decode_per_kv_ms = c.attn_decode_per_kv_ms;
    p.fixed_overhead_ms = c.fixed_overhead_ms;
    p.tp_comm_ms = c.tp_comm_ms;
    p.pp_send_ms = c.pp_send_ms;
    p.tile_size = c.tile_size;
    p.tile_penalty_frac = c.tile_penalty_frac;
    return p;
}

int code_of(const std::exception& e) {
    if (dynamic_cast<const OutOfKvBlocks*>(&e)) return 2;
    if (dynamic_cast<const InfeasibleSlo*>(&e)) return 3;
    if (dynamic_cast<const ContractViolation*>(&e)) return 1;
    return 7;
}

}  // namespace

struct ref_report {
    SimReport rep;
    std::string jsonl;
};

extern "C" {

int ref_cost_preset(const char* name, ssh_cost_params* out) {
    auto p = model_preset(name);
    if (!p) return 1;
    out->per_token_linear_ms = p->per_token_linear_ms;
    out->saturation_tokens = p->saturation_tokens;
    out->attn_prefill_quad_ms = p->attn_prefill_quad_ms;
    out->attn_kv_read_ms = p->attn_kv_read_ms;
    out->attn_decode_per_kv_ms = p->attn_decode_per_kv_ms;
    out->fixed_overhead_ms = p->fixed_overhead_ms;
    out->tp_comm_ms = p->tp_comm_ms;
    out->pp_send_ms = p->pp_send_ms;
    out->tile_size = p->tile_size;
    out->tile_penalty_frac = p->tile_penalty_frac;
    return 0;
}

int ref_make_trace(const char* workload, double qps, int n, uint64_t seed, ssh_request* out) {
    try {
        auto w = workload_preset(workload);
        if (!w) return 1;
        auto t = make_trace(*w, qps, n, seed);
        for (int i = 0; i < n; ++i) out[i] = ssh_request{t[i].arrival_time, t[i].prompt_tokens, t[i].output_tokens};
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

int ref_simulate(const ssh_replica_cfg* cfg, const ssh_cost_params* params, const ssh_request* trace, int n,
                 ref_report** out) {
    try {
        std::vector<Request> reqs;
        for (int i = 0; i < n; ++i) reqs.emplace_back(i, trace[i].arrival_us, trace[i].prompt_tokens, trace[i].output_tokens);
        auto* r = new ref_report();
        try {
            r->rep = simulate(to_cfg(*cfg), to_params(*params), reqs);
        } catch (...) {
            delete r;
            throw;
        }
        r->jsonl = r->rep.event_log_jsonl();
        *out = r;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

const char* ref_report_event_log(ref_report* r, size_t* len) {
    *len = r->jsonl.size();
    return r->jsonl.c_str();
}

int ref_summary(ref_report* r, double warmup, ssh_latency* out) {
    const LatencyReport L = summarize(r->rep, warmup);
    *out = ssh_latency{L.ttft_median_ms, L.tbt_p99_ms, L.tbt_median_ms, L.sched_delay_median_ms,
                       L.throughput_tps, L.bubble_fraction, L.makespan_ms, L.tbt_samples, L.n_requests};
    return 0;
}

void ref_report_free(ref_report* r) { delete r; }

double ref_iteration_time(const ssh_entry* e, int n, const ssh_cost_params* p, int tp, int pp) {
    Batch b;
    for (int i = 0; i < n; ++i) {
        BatchEntry be;
        be.request_id = e[i].request_id;
        be.kind = e[i].kind ? EntryKind::PrefillChunk : EntryKind::Decode;
        be.chunk_tokens = e[i].chunk_tokens;
        be.prefix_tokens = e[i].prefix_tokens;
        b.entries.push_back(be);
    }
    return iteration_time(b, to_params(*p), tp, pp);
}

int ref_token_budget(double t_max_ms, const ssh_cost_params* p, int pp, int* out) {
    try {
        *out = compute_token_budget(t_max_ms, to_params(*p), pp);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

// Same argument layout as ssh_calibrate; returns 0, or 8 with the reference's
// CalibrationError message in ref_last_error().
int ref_calibrate(const ssh_anchor* anchors, int n, const ssh_calib_opts* opts, ssh_cost_params* out,
                  double* predicted_ms, double* max_rel, int* zeroed_mask) {
    try {
        std::vector<CalibrationAnchor> an;
        for (int i = 0; i < n; ++i) {
            Batch b;
            for (int j = 0; j < anchors[i].n_entries; ++j) {
                const ssh_entry& e = anchors[i].entries[j];
                BatchEntry be;
                be.request_id = e.request_id;
                be.kind = e.kind ? EntryKind::PrefillChunk : EntryKind::Decode;
                be.chunk_tokens = e.chunk_tokens;
                be.prefix_tokens = e.prefix_tokens;
                b.entries.push_back(be);
            }
            an.push_back(CalibrationAnchor{b, anchors[i].observed_ms});
        }
        CalibrationOptions o;
        if (opts) {
            o.tile_size = opts->tile_size;
            o.tile_penalty_frac = opts->tile_penalty_frac;
            o.max_saturation_tokens = opts->max_saturation_tokens;
        }
        const CalibrationResult r = calibrate(an, o);
        const CostModelParams& q = r.params;
        *out = ssh_cost_params{q.per_token_linear_ms, q.saturation_tokens, q.attn_prefill_quad_ms, q.attn_kv_read_ms,
                               q.attn_decode_per_kv_ms, q.fixed_overhead_ms, q.tp_comm_ms, q.pp_send_ms,
                               q.tile_size, q.tile_penalty_frac};
        for (int i = 0; i < n; ++i)
            if (predicted_ms) predicted_ms[i] = r.predicted_ms[size_t(i)];
        if (max_rel) *max_rel = r.max_relative_error;
        if (zeroed_mask) {
            static const char* const names[5] = {"fixed_overhead_ms", "per_token_linear_ms", "attn_prefill_quad_ms",
                                                 "attn_kv_read_ms", "attn_decode_per_kv_ms"};
            int m = 0;
            for (const auto& z : r.zeroed_terms)
                for (int t = 0; t < 5; ++t)
                    if (z == names[t]) m |= 1 << t;
            *zeroed_mask = m;
        }
        return 0;
    } catch (const CalibrationError& e) {
        g_err = e.what();
        return 8;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

// Same layout as ssh_capacity_search (no GPU). The reference is built here
// without OpenMP, so its ladder probes one rung at a time (opts->parallel unused).
int ref_capacity(const ssh_replica_cfg* cfg, const ssh_cost_params* params, const char* workload, int probe_requests,
                 uint64_t seed, double slo_ms, const ssh_capacity_opts* opts, double* qps_out, int* monotone,
                 ssh_capacity_probe* probes, int cap, int* n_probes) {
    try {
        const auto w = workload_preset(workload);
        if (!w) throw ContractViolation("unknown workload preset");
        const ReplicaConfig rc = to_cfg(*cfg);
        const CostModelParams cp = to_params(*params);
        CapacityOptions o;
        o.qps_low = opts->qps_low;
        o.max_qps = opts->max_qps;
        o.rel_width = opts->rel_width;
        const ProbeFn probe = [&](double qps) {
            SimOptions so;
            so.keep_events = false;
            so.keep_microbatches = false;
            so.keep_kv_series = false;
            return summarize(simulate(rc, cp, make_trace(*w, qps, probe_requests, seed), so));
        };
        const CapacityResult r = capacity_search(probe, slo_ms, o);
        *qps_out = r.qps;
        *monotone = r.monotone_warning;
        *n_probes = int(r.probes.size());
        for (size_t i = 0; i < r.probes.size() && int(i) < cap; ++i) {
            const LatencyReport& L = r.probes[i].report;
            probes[i] = ssh_capacity_probe{r.probes[i].qps, r.probes[i].pass,
                                           ssh_latency{L.ttft_median_ms, L.tbt_p99_ms, L.tbt_median_ms,
                                                       L.sched_delay_median_ms, L.throughput_tps,
                                                       L.bubble_fraction, L.makespan_ms, L.tbt_samples,
                                                       L.n_requests}};
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

double ref_decode_reference_time(const ssh_cost_params* p) { return decode_reference_time(to_params(*p)); }

const char* ref_last_error(void) { return g_err.c_str(); }

}  // extern "C"
