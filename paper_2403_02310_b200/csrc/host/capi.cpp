// extern "C" surface of the host engine (include/ss_host.h) and the GPU
// executor that plugs ss_forward_hybrid into the engine's model step.
#include <cstring>
#include <memory>
#include <string>

#include "../../../include/ss_host.h"
#include "calibrate.hpp"
#include "capacity.hpp"
#include "costmodel.hpp"
#include "descriptor.hpp"
#include "engine.hpp"
#include "metrics.hpp"
#include "sched.hpp"
#include "workload.hpp"

struct ssh_report {
    ss::Report rep;
    std::string jsonl;
    bool jsonl_ready = false;
};

struct ssh_session {
    ss::KvLedger kv;
    int32_t vocab;
    std::uint64_t seed;
    ssh_session(std::int64_t blocks, std::int32_t bs, std::int32_t v, std::uint64_t sd) : kv(blocks, bs), vocab(v), seed(sd) {}
};

struct ssh_desc {
    ss::HostDesc d;
    ss_batch_desc view;
    std::int64_t pool_blocks = 0;
};

namespace {

thread_local std::string g_err;

template <class F>
ss_status guarded(F&& f) {
    try {
        f();
        return SS_OK;
    } catch (const ss::OutOfKvBlocks& e) {
        g_err = e.what();
        return SS_OUT_OF_KV;
    } catch (const ss::InfeasibleSlo& e) {
        g_err = e.what();
        return SS_INFEASIBLE;
    } catch (const ss::CalibrationError& e) {
        g_err = e.what();
        return SS_CALIBRATION;
    } catch (const ss::ContractViolation& e) {
        g_err = e.what();
        return SS_INVALID_ARG;
    } catch (const std::bad_alloc& e) {
        g_err = e.what();
        return SS_OUT_OF_MEMORY;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SS_INTERNAL;
    }
}

ss::ReplicaConfig to_cfg(const ssh_replica_cfg& c) {
    ss::ReplicaConfig r;
    if (c.scheduler < 0 || c.scheduler > 3) throw ss::ContractViolation("unknown scheduler policy");
    r.policy = ss::Policy(c.scheduler);
    r.token_budget = c.token_budget;
    r.max_batch_size = c.max_batch_size;
    r.max_num_batched_tokens = c.max_num_batched_tokens;
    r.max_batch_size_orca = c.max_batch_size_orca;
    r.tp = c.tp_degree;
    r.pp = c.pp_degree;
    r.kv_blocks = c.kv_blocks;
    r.block_size = c.kv_block_size;
    r.tile_size = c.tile_size;
    r.chunk_align = c.chunk_align;
    r.reserve_decode_tokens = c.reserve_decode_tokens;
    r.watermark = c.kv_watermark_frac;
    r.pipeline_tbt_factor = c.pipeline_tbt_factor;
    r.hybrid_batching = c.hybrid_batching != 0;
    return r;
}

ss::CostParams to_params(const ssh_cost_params& c) {
    ss::CostParams p;
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

ss::Batch to_batch(const ssh_entry* e, int32_t n) {
    ss::Batch b;
    for (int32_t i = 0; i < n; ++i)
        b.entries.push_back(ss::Entry{e[i].request_id, e[i].kind ? ss::Kind::Chunk : ss::Kind::Decode,
                                      e[i].chunk_tokens, e[i].prefix_tokens});
    return b;
}

// Model step = one real forward on the GPU (replaces iteration_time at
// engine.cpp:227). Time is the library's CUDA-event measurement.
class GpuExecutor final : public ss::StepExecutor {
public:
    // The GPU step is one whole-model forward on this rank's TP shard: the replica must be
    // un-pipelined (the reference divides iteration_time by pp, costmodel.cpp:55; a GPU
    // pipeline is not built) and its tp degree must be the context's (every rank runs the
    // same replicated schedule).
    GpuExecutor(ss_ctx* ctx, std::uint64_t seed, const ss::ReplicaConfig& rc) : ctx_(ctx), seed_(seed) {
        ss_model_cfg mc;
        int32_t r, t;
        if (ss_model_config(ctx, &mc, &r, &t) != SS_OK) throw ss::ContractViolation("invalid GPU context");
        if (rc.pp != 1)
            throw ss::ContractViolation("GPU model step: pp_degree must be 1 (the forward covers all layers)");
        if (rc.tp != t)
            throw ss::ContractViolation("GPU model step: tp_degree " + std::to_string(rc.tp) +
                                        " differs from the GPU context's tp_size " + std::to_string(t));
        vocab_ = mc.vocab;
    }
    double step_ms(const ss::Batch& b, const ss::KvLedger& kv, const std::vector<ss::Request>& reqs) override {
        const ss::HostDesc d = ss::build_desc(b, kv, reqs, seed_, vocab_);
        const ss_batch_desc v = d.view();
        float ms = 0.f;
        const ss_status st = ss_forward_hybrid(ctx_, &v, nullptr, nullptr, &ms);
        if (st == SS_OUT_OF_KV) throw ss::OutOfKvBlocks(std::string("GPU forward: ") + ss_last_error(ctx_));
        if (st != SS_OK) throw std::runtime_error(std::string("GPU forward failed: ") + ss_last_error(ctx_));
        return double(ms);
    }

private:
    ss_ctx* ctx_;
    std::uint64_t seed_;
    int32_t vocab_ = 0;
};

// Pipeline-parallel model step: the batch runs through every stage (ss_forward_pipeline); the
// engine's pipeline model (engine.cpp:42-81) takes one per-stage time per micro-batch, the
// reference's iteration_time / pp (costmodel.cpp:55): here the slowest stage's measured time.
class GpuPipelineExecutor final : public ss::StepExecutor {
public:
    GpuPipelineExecutor(ss_ctx* const* stages, int32_t n, std::uint64_t seed, const ss::ReplicaConfig& rc)
        : stages_(stages, stages + n), seed_(seed), ms_(size_t(n)) {
        if (n < 2 || rc.pp != n)
            throw ss::ContractViolation("GPU pipeline: pp_degree must equal the number of stage contexts (>= 2)");
        if (rc.tp != 1) throw ss::ContractViolation("GPU pipeline: tp_degree must be 1");
        ss_model_cfg mc;
        int32_t r, t;
        if (ss_model_config(stages[0], &mc, &r, &t) != SS_OK) throw ss::ContractViolation("invalid GPU context");
        vocab_ = mc.vocab;
    }
    double step_ms(const ss::Batch& b, const ss::KvLedger& kv, const std::vector<ss::Request>& reqs) override {
        const ss::HostDesc d = ss::build_desc(b, kv, reqs, seed_, vocab_);
        const ss_batch_desc v = d.view();
        const ss_status st = ss_forward_pipeline(stages_.data(), int32_t(stages_.size()), &v, nullptr, nullptr, ms_.data());
        if (st == SS_OUT_OF_KV) throw ss::OutOfKvBlocks(std::string("GPU forward: ") + ss_last_error(stages_.back()));
        if (st != SS_OK) throw std::runtime_error(std::string("GPU pipeline forward failed: ") + ss_last_error(stages_.back()));
        double worst = 0.0;
        for (float x : ms_) worst = std::max(worst, double(x));
        return worst;
    }

private:
    std::vector<ss_ctx*> stages_;
    std::uint64_t seed_;
    std::vector<float> ms_;
    int32_t vocab_ = 0;
};

std::unique_ptr<ss::StepExecutor> make_executor(ss_ctx* gpu, ss_ctx* const* stages, int32_t n_stages,
                                                std::uint64_t token_seed, const ss::ReplicaConfig& rc,
                                                const ss::CostParams& cp) {
    if (gpu && n_stages > 0) throw ss::ContractViolation("set either gpu or gpu_stages");
    if (n_stages > 0) return std::make_unique<GpuPipelineExecutor>(stages, n_stages, token_seed, rc);
    if (gpu) return std::make_unique<GpuExecutor>(gpu, token_seed, rc);
    return std::make_unique<ss::CostModelExecutor>(cp, rc.tp, rc.pp);
}

ssh_desc* make_desc(const ss::Batch& b, const std::vector<bool>& completes, int32_t bs, int32_t vocab,
                    std::uint64_t seed) {
    if (vocab < 1) throw ss::ContractViolation("vocab must be >= 1");
    std::int64_t need = 0;
    for (const ss::Entry& e : b.entries) need += ss::blocks_for(e.prefix + e.tokens, bs);
    ss::KvLedger kv(need, bs);
    for (const ss::Entry& e : b.entries) {
        if (kv.live(e.rid)) throw ss::ContractViolation("duplicate request id in explicit batch");
        kv.admit(e.rid, e.prefix + e.tokens);
        kv.grow(e.rid, e.prefix + e.tokens);
    }
    auto out = std::make_unique<ssh_desc>();
    out->d = ss::build_desc(b, kv, completes, seed, vocab);
    out->view = out->d.view();
    out->pool_blocks = kv.peak_allocated();
    return out.release();
}

}  // namespace

extern "C" {

void ssh_replica_default(ssh_replica_cfg* out) {
    const ss::ReplicaConfig d;
    out->scheduler = int32_t(d.policy);
    out->token_budget = d.token_budget;
    out->max_batch_size = d.max_batch_size;
    out->max_num_batched_tokens = d.max_num_batched_tokens;
    out->max_batch_size_orca = d.max_batch_size_orca;
    out->tp_degree = d.tp;
    out->pp_degree = d.pp;
    out->kv_blocks = d.kv_blocks;
    out->kv_block_size = d.block_size;
    out->tile_size = d.tile_size;
    out->chunk_align = d.chunk_align;
    out->reserve_decode_tokens = d.reserve_decode_tokens;
    out->kv_watermark_frac = d.watermark;
    out->pipeline_tbt_factor = d.pipeline_tbt_factor;
    out->hybrid_batching = d.hybrid_batching ? 1 : 0;
}

ss_status ssh_cost_preset(const char* name, ssh_cost_params* out) {
    return guarded([&] {
        const auto p = ss::cost_preset(name ? name : "");
        if (!p) throw ss::ContractViolation(std::string("unknown model preset: ") + (name ? name : "(null)"));
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
    });
}

static void copy_trace(const std::vector<ss::Request>& t, ssh_request* out) {
    for (std::size_t i = 0; i < t.size(); ++i) out[i] = ssh_request{t[i].arrival, t[i].prompt, t[i].output};
}

ss_status ssh_make_trace(const char* workload, double qps, int32_t n, uint64_t seed, ssh_request* out) {
    return guarded([&] {
        const auto w = ss::workload_preset(workload ? workload : "");
        if (!w) throw ss::ContractViolation("unknown workload preset");
        copy_trace(ss::make_trace(*w, qps, n, seed), out);
    });
}

ss_status ssh_make_trace_spec(double pm, double p90, double om, double o90, int64_t max_total, double qps,
                              int32_t n, uint64_t seed, ssh_request* out) {
    return guarded([&] {
        ss::WorkloadSpec w{"custom", {pm, p90}, {om, o90}, max_total};
        copy_trace(ss::make_trace(w, qps, n, seed), out);
    });
}

ss_status ssh_simulate(const ssh_replica_cfg* cfg, const ssh_cost_params* params, const ssh_request* trace,
                       int32_t n, const ssh_sim_opts* opts, ssh_report** out) {
    return guarded([&] {
        if (!cfg || !params || (!trace && n > 0) || !out) throw ss::ContractViolation("null argument");
        std::vector<ss::Request> reqs;
        for (int32_t i = 0; i < n; ++i) reqs.emplace_back(i, trace[i].arrival_us, trace[i].prompt_tokens, trace[i].output_tokens);
        ss::SimOptions so;
        ss_ctx* gpu = nullptr;
        ss_ctx* const* stages = nullptr;
        int32_t n_stages = 0;
        std::uint64_t token_seed = 0;
        if (opts) {
            so.keep_events = opts->keep_events != 0;
            if (opts->max_events > 0) so.max_events = opts->max_events;
            so.check_block_tables = opts->check_block_tables != 0;
            gpu = opts->gpu;
            stages = opts->gpu_stages;
            n_stages = opts->gpu_stages ? opts->n_gpu_stages : 0;
            token_seed = opts->token_seed;
        }
        const ss::ReplicaConfig rc = to_cfg(*cfg);
        const ss::CostParams cp = to_params(*params);
        std::unique_ptr<ss::StepExecutor> exec = make_executor(gpu, stages, n_stages, token_seed, rc, cp);
        auto r = std::make_unique<ssh_report>();
        r->rep = ss::simulate(rc, cp, reqs, *exec, so);
        *out = r.release();
    });
}

const char* ssh_report_event_log(ssh_report* r, size_t* len) {
    if (!r) return nullptr;
    if (!r->jsonl_ready) {
        r->jsonl = r->rep.event_log_jsonl();
        r->jsonl_ready = true;
    }
    if (len) *len = r->jsonl.size();
    return r->jsonl.c_str();
}

ss_status ssh_report_summary(const ssh_report* r, double warmup_frac, ssh_latency* out) {
    return guarded([&] {
        const ss::Latency L = ss::summarize(r->rep, warmup_frac);
        *out = ssh_latency{L.ttft_median_ms, L.tbt_p99_ms, L.tbt_median_ms, L.sched_delay_median_ms,
                           L.throughput_tps, L.bubble_fraction, L.makespan_ms, L.tbt_samples, L.n_requests};
    });
}

int64_t ssh_report_num_microbatches(const ssh_report* r) { return r ? int64_t(r->rep.mbs.size()) : 0; }

int32_t ssh_report_microbatch(const ssh_report* r, int64_t i, ssh_entry* out, int32_t cap, double* iteration_ms,
                              int64_t* issue_us) {
    if (!r || i < 0 || i >= int64_t(r->rep.mbs.size())) return -1;
    const ss::MbRecord& mb = r->rep.mbs[std::size_t(i)];
    for (std::size_t k = 0; k < mb.entries.size() && int32_t(k) < cap; ++k) {
        const ss::Entry& e = mb.entries[k];
        out[k] = ssh_entry{e.rid, int32_t(e.kind), e.tokens, e.prefix};
    }
    if (iteration_ms) *iteration_ms = mb.iteration_ms;
    if (issue_us) *issue_us = mb.issue;
    return int32_t(mb.entries.size());
}

int64_t ssh_report_peak_blocks(const ssh_report* r) { return r ? r->rep.peak_blocks : 0; }

void ssh_report_free(ssh_report* r) { delete r; }

double ssh_iteration_time(const ssh_entry* entries, int32_t n, const ssh_cost_params* p, int32_t tp, int32_t pp) {
    return ss::iteration_time(to_batch(entries, n), to_params(*p), tp, pp);
}

double ssh_decode_reference_time(const ssh_cost_params* p) { return ss::decode_reference_time(to_params(*p)); }

ss_status ssh_calibrate(const ssh_anchor* anchors, int32_t n, const ssh_calib_opts* opts, ssh_cost_params* out,
                        double* predicted_ms, double* relative_error, double* max_relative_error,
                        int32_t* zeroed_mask) {
    return guarded([&] {
        if (!out || n < 0 || (n > 0 && !anchors)) throw ss::ContractViolation("null calibration argument");
        std::vector<ss::Anchor> an;
        for (int32_t i = 0; i < n; ++i) {
            if (anchors[i].n_entries > 0 && !anchors[i].entries) throw ss::ContractViolation("null anchor entries");
            an.push_back(ss::Anchor{to_batch(anchors[i].entries, anchors[i].n_entries), anchors[i].observed_ms});
        }
        ss::CalibrationOptions o;
        if (opts) {
            o.tile_size = opts->tile_size;
            o.tile_penalty_frac = opts->tile_penalty_frac;
            o.max_saturation_tokens = opts->max_saturation_tokens;
        }
        const ss::Calibration c = ss::calibrate(an, o);
        ssh_cost_params r{};
        r.per_token_linear_ms = c.params.per_token_linear_ms;
        r.saturation_tokens = c.params.saturation_tokens;
        r.attn_prefill_quad_ms = c.params.attn_prefill_quad_ms;
        r.attn_kv_read_ms = c.params.attn_kv_read_ms;
        r.attn_decode_per_kv_ms = c.params.attn_decode_per_kv_ms;
        r.fixed_overhead_ms = c.params.fixed_overhead_ms;
        r.tp_comm_ms = c.params.tp_comm_ms;
        r.pp_send_ms = c.params.pp_send_ms;
        r.tile_size = c.params.tile_size;
        r.tile_penalty_frac = c.params.tile_penalty_frac;
        *out = r;
        for (int32_t i = 0; i < n; ++i) {
            if (predicted_ms) predicted_ms[i] = c.predicted_ms[size_t(i)];
            if (relative_error) relative_error[i] = c.relative_error[size_t(i)];
        }
        if (max_relative_error) *max_relative_error = c.max_relative_error;
        if (zeroed_mask) {
            static const char* const names[5] = {"fixed_overhead_ms", "per_token_linear_ms", "attn_prefill_quad_ms",
                                                 "attn_kv_read_ms", "attn_decode_per_kv_ms"};
            int32_t m = 0;
            for (const std::string& z : c.zeroed_terms)
                for (int t = 0; t < 5; ++t)
                    if (z == names[t]) m |= 1 << t;
            *zeroed_mask = m;
        }
    });
}

ss_status ssh_capacity_search(const ssh_replica_cfg* cfg, const ssh_cost_params* params, const char* workload,
                              int32_t probe_requests, uint64_t seed, double slo_ms, const ssh_capacity_opts* opts,
                              const ssh_sim_opts* sim, double* qps_out, int32_t* monotone_warning,
                              ssh_capacity_probe* probes, int32_t cap, int32_t* n_probes) {
    return guarded([&] {
        if (!cfg || !params || !qps_out) throw ss::ContractViolation("null argument");
        const auto w = ss::workload_preset(workload ? workload : "");
        if (!w) throw ss::ContractViolation("unknown workload preset");
        const ss::ReplicaConfig rc = to_cfg(*cfg);
        const ss::CostParams cp = to_params(*params);
        ss::CapacityOptions o;
        if (opts) {
            o.qps_low = opts->qps_low;
            o.max_qps = opts->max_qps;
            o.rel_width = opts->rel_width;
            o.parallel = opts->parallel;
        }
        ss_ctx* gpu = sim ? sim->gpu : nullptr;
        ss_ctx* const* stages = sim ? sim->gpu_stages : nullptr;
        const int32_t n_stages = stages ? sim->n_gpu_stages : 0;
        if ((gpu || n_stages) && o.parallel != 1)
            throw ss::ContractViolation("GPU capacity probes run one at a time (parallel = 1)");
        const std::uint64_t token_seed = sim ? sim->token_seed : 0;
        const ss::Probe probe = [&](double qps) {
            const std::vector<ss::Request> trace = ss::make_trace(*w, qps, probe_requests, seed);
            ss::SimOptions so;
            so.keep_events = false;  // probe_sim_options, cli.cpp:373-379
            std::unique_ptr<ss::StepExecutor> exec = make_executor(gpu, stages, n_stages, token_seed, rc, cp);
            return ss::summarize(ss::simulate(rc, cp, trace, *exec, so));
        };
        const ss::CapacityResult r = ss::capacity_search(probe, slo_ms, o);
        *qps_out = r.qps;
        if (monotone_warning) *monotone_warning = r.monotone_warning;
        if (n_probes) *n_probes = int32_t(r.probes.size());
        for (std::size_t i = 0; probes && i < r.probes.size() && int32_t(i) < cap; ++i) {
            const ss::Latency& L = r.probes[i].report;
            probes[i] = ssh_capacity_probe{r.probes[i].qps, r.probes[i].pass,
                                           ssh_latency{L.ttft_median_ms, L.tbt_p99_ms, L.tbt_median_ms,
                                                       L.sched_delay_median_ms, L.throughput_tps, L.bubble_fraction,
                                                       L.makespan_ms, L.tbt_samples, L.n_requests}};
        }
    });
}

ss_status ssh_compute_token_budget(double t_max_ms, const ssh_cost_params* p, int32_t pp, int32_t* out) {
    return guarded([&] { *out = ss::token_budget_for(t_max_ms, to_params(*p), pp); });
}

int32_t ssh_next_chunk_size(int32_t prompt, int32_t prefill_done, int32_t budget, int32_t packed, int32_t align) {
    ss::Request r(0, 0, prompt, 1);
    r.prefill_done = prefill_done;
    return ss::next_chunk(r, budget, packed, align);
}

ss_status ssh_percentile(const double* series, int64_t n, double p, double* out) {
    return guarded([&] { *out = ss::percentile(std::vector<double>(series, series + n), p); });
}

ss_status ssh_desc_build(const ssh_entry* entries, int32_t n, const int32_t* completes, int32_t bs, int32_t vocab,
                         uint64_t seed, ssh_desc** out) {
    return guarded([&] {
        ss::Batch b = to_batch(entries, n);
        std::vector<bool> c;
        for (int32_t i = 0; i < n; ++i) c.push_back(completes ? completes[i] != 0 : true);
        *out = make_desc(b, c, bs, vocab, seed);
    });
}

ss_status ssh_desc_canonical(int32_t tau, int32_t n_dec, int64_t kv_each, int64_t chunk_prefix, int32_t bs,
                             int32_t vocab, uint64_t seed, ssh_desc** out) {
    return guarded([&] {
        if (tau - n_dec < 1) throw ss::ContractViolation("token budget leaves no room for the chunk");
        ss::Batch b = ss::canonical_batch(tau, n_dec, kv_each, chunk_prefix);
        *out = make_desc(b, std::vector<bool>(b.entries.size(), true), bs, vocab, seed);
    });
}

ss_status ssh_session_create(int64_t kv_blocks, int32_t bs, int32_t vocab, uint64_t seed, ssh_session** out) {
    return guarded([&] {
        if (vocab < 1) throw ss::ContractViolation("vocab must be >= 1");
        *out = new ssh_session(kv_blocks, bs, vocab, seed);
    });
}

ss_status ssh_session_step(ssh_session* s, const ssh_entry* entries, int32_t n, const int32_t* prompt_lens,
                           ssh_desc** out) {
    return guarded([&] {
        if (!s || !entries || n < 1 || !prompt_lens || !out) throw ss::ContractViolation("null argument");
        ss::Batch b = to_batch(entries, n);
        std::vector<bool> completes;
        for (int32_t i = 0; i < n; ++i) {
            const ss::Entry& e = b.entries[std::size_t(i)];
            if (!s->kv.live(e.rid)) s->kv.admit(e.rid, prompt_lens[i]);
            s->kv.grow(e.rid, e.prefix + e.tokens);
            completes.push_back(e.kind == ss::Kind::Chunk && e.prefix + e.tokens == prompt_lens[i]);
        }
        auto d = std::make_unique<ssh_desc>();
        d->d = ss::build_desc(b, s->kv, completes, s->seed, s->vocab);
        d->view = d->d.view();
        d->pool_blocks = s->kv.peak_allocated();
        *out = d.release();
    });
}

ss_status ssh_session_release(ssh_session* s, int32_t rid) {
    return guarded([&] { s->kv.release(rid); });
}

int64_t ssh_session_peak_blocks(const ssh_session* s) { return s ? s->kv.peak_allocated() : 0; }
void ssh_session_free(ssh_session* s) { delete s; }

const ss_batch_desc* ssh_desc_view(const ssh_desc* d) { return d ? &d->view : nullptr; }
int64_t ssh_desc_pool_blocks(const ssh_desc* d) { return d ? d->pool_blocks : 0; }
void ssh_desc_free(ssh_desc* d) { delete d; }

const char* ssh_last_error(void) { return g_err.c_str(); }

}  // extern "C"
