/*
 * ss_host.h — C ABI of the host-side engine (scheduler, KV ledger + block
 * tables, discrete-event engine, trace synthesis, latency summary).
 *
 * This is the B200 framework's restatement of the reference simulator's host
 * path (servesim). Every entry point names the reference symbol whose
 * semantics it reproduces bit for bit; the only behavioural addition is that
 * the engine's model step can be a real GPU forward (ss_gpu.h) instead of the
 * analytical cost model.
 *
 *   ssh_simulate          <- servesim::simulate            engine.cpp:326-330
 *   ssh_report_event_log  <- SimReport::event_log_jsonl    engine.cpp:332-371
 *   ssh_report_summary    <- servesim::summarize           metrics.cpp:23-59
 *   ssh_make_trace        <- servesim::make_trace          workload.cpp:73-84
 *   ssh_iteration_time    <- servesim::iteration_time      costmodel.cpp:39-56
 *   ssh_compute_token_budget <- compute_token_budget       sched.cpp:154-175
 *   ssh_next_chunk_size   <- get_next_chunk_size           sched.cpp:97-103
 *   ssh_percentile        <- percentile                    metrics.cpp:13-21
 *   ssh_decode_reference_time <- decode_reference_time     costmodel.cpp:83-85
 *   ssh_calibrate         <- servesim::calibrate           calibrate.cpp:121-193
 *   ssh_capacity_search   <- servesim::capacity_search     metrics.cpp:70-138
 *                            (probe = make_trace + simulate + summarize, cli.cpp:434-439)
 *
 * No exceptions cross this boundary: every call returns an ss_status and the
 * message of the last failure is available from ssh_last_error().
 */
#ifndef SS_HOST_H
#define SS_HOST_H

#include <stddef.h>
#include <stdint.h>

#include "ss_gpu.h"
#include "ss_status.h"

#ifdef __cplusplus
extern "C" {
#endif

/* servesim::SchedulerPolicy (core.hpp:99) */
enum { SSH_REQUEST_LEVEL = 0, SSH_VLLM = 1, SSH_ORCA = 2, SSH_STALL_FREE = 3 };

/* servesim::ReplicaConfig (core.hpp:105-125); ssh_replica_default() gives the
 * reference defaults. */
typedef struct {
    int32_t scheduler;
    int32_t token_budget;
    int32_t max_batch_size;
    int32_t max_num_batched_tokens;
    int32_t max_batch_size_orca;
    int32_t tp_degree;
    int32_t pp_degree;
    int64_t kv_blocks;
    int32_t kv_block_size;
    int32_t tile_size;
    int32_t chunk_align;
    int32_t reserve_decode_tokens;
    double kv_watermark_frac;
    double pipeline_tbt_factor;
    int32_t hybrid_batching;
} ssh_replica_cfg;

/* servesim::CostModelParams (costmodel.hpp:19-41) */
typedef struct {
    double per_token_linear_ms;
    int32_t saturation_tokens;
    double attn_prefill_quad_ms;
    double attn_kv_read_ms;
    double attn_decode_per_kv_ms;
    double fixed_overhead_ms;
    double tp_comm_ms;
    double pp_send_ms;
    int32_t tile_size;
    double tile_penalty_frac;
} ssh_cost_params;

/* One trace row: servesim::Request's immutable fields (core.hpp:40-61). */
typedef struct {
    int64_t arrival_us;
    int32_t prompt_tokens;
    int32_t output_tokens;
} ssh_request;

/* servesim::BatchEntry (core.hpp:73-78); kind 0 = decode, 1 = prefill chunk. */
typedef struct {
    int32_t request_id;
    int32_t kind;
    int32_t chunk_tokens;
    int64_t prefix_tokens;
} ssh_entry;

/* servesim::LatencyReport (metrics.hpp:12-22) */
typedef struct {
    double ttft_median_ms;
    double tbt_p99_ms;
    double tbt_median_ms;
    double sched_delay_median_ms;
    double throughput_tps;
    double bubble_fraction;
    double makespan_ms;
    int64_t tbt_samples;
    int32_t n_requests;
} ssh_latency;

/* Options of one simulation. gpu == NULL runs the reference cost model as the
 * model step; otherwise every issued batch is executed by ss_forward_hybrid on
 * that context and the measured GPU time replaces iteration_time()
 * (engine.cpp:227). token_seed seeds the synthetic token ids fed to the GPU. */
typedef struct {
    int32_t keep_events;
    int64_t max_events;
    ss_ctx* gpu;
    uint64_t token_seed;
    int32_t check_block_tables; /* assert block counts == ledger counts each issue */
    /* pipeline-parallel model step (pp_degree == n_gpu_stages > 1): gpu_stages[i] is
     * stage i (ss_create_pp_stage); every issued batch runs ss_forward_pipeline and
     * the slowest stage's device time is the per-stage time of the reference's
     * pipeline model (engine.cpp:42-81). gpu must then be NULL. */
    ss_ctx* const* gpu_stages;
    int32_t n_gpu_stages;
} ssh_sim_opts;

typedef struct ssh_report ssh_report;

void ssh_replica_default(ssh_replica_cfg* out);
/* name in {"mistral7b","yi34b","llama70b","falcon180b","tiny"}; "tiny" is the
 * test clock of test_engine.cpp:14-25. */
ss_status ssh_cost_preset(const char* name, ssh_cost_params* out);

ss_status ssh_make_trace(const char* workload, double qps, int32_t n, uint64_t seed,
                         ssh_request* out /* n rows */);
/* Explicit (median, p90) log-normal spec, workload.hpp:31-47. */
ss_status ssh_make_trace_spec(double prompt_median, double prompt_p90, double output_median,
                              double output_p90, int64_t max_total, double qps, int32_t n,
                              uint64_t seed, ssh_request* out);

ss_status ssh_simulate(const ssh_replica_cfg* cfg, const ssh_cost_params* params,
                       const ssh_request* trace, int32_t n, const ssh_sim_opts* opts,
                       ssh_report** out);
/* Pointer stays valid until ssh_report_free. */
const char* ssh_report_event_log(ssh_report* r, size_t* len);
ss_status ssh_report_summary(const ssh_report* r, double warmup_frac, ssh_latency* out);
int64_t ssh_report_num_microbatches(const ssh_report* r);
/* Micro-batch i: entries (copied into out up to cap), measured/modelled ms. */
int32_t ssh_report_microbatch(const ssh_report* r, int64_t i, ssh_entry* out, int32_t cap,
                              double* iteration_ms, int64_t* issue_us);
/* Peak number of KV blocks simultaneously allocated over the run. */
int64_t ssh_report_peak_blocks(const ssh_report* r);
void ssh_report_free(ssh_report* r);

double ssh_iteration_time(const ssh_entry* entries, int32_t n, const ssh_cost_params* p,
                          int32_t tp, int32_t pp);
double ssh_decode_reference_time(const ssh_cost_params* p);
ss_status ssh_compute_token_budget(double t_max_ms, const ssh_cost_params* p, int32_t pp_degree,
                                   int32_t* out_budget);
/* servesim::CalibrationAnchor (costmodel.hpp:78-81): a batch + its observed ms. */
typedef struct {
    const ssh_entry* entries;
    int32_t n_entries;
    double observed_ms;
} ssh_anchor;

/* servesim::CalibrationOptions (costmodel.hpp:91-95); NULL = the defaults
 * (tile 256, penalty 0.32, saturation swept over 1..2048). */
typedef struct {
    int32_t tile_size;
    double tile_penalty_frac;
    int32_t max_saturation_tokens;
} ssh_calib_opts;

/* servesim::calibrate (calibrate.cpp:121-193): fits the cost-model constants to
 * observed timings (e.g. B200 forwards of anchor batches). predicted_ms and
 * relative_error (nullable) receive n values; zeroed_mask (nullable) gets bit t
 * set for every term pinned to zero, t in order (fixed_overhead, per_token_linear,
 * attn_prefill_quad, attn_kv_read, attn_decode_per_kv). SS_CALIBRATION carries
 * the reference's CalibrationError message. */
ss_status ssh_calibrate(const ssh_anchor* anchors, int32_t n, const ssh_calib_opts* opts,
                        ssh_cost_params* out, double* predicted_ms, double* relative_error,
                        double* max_relative_error, int32_t* zeroed_mask);
/* servesim::CapacityOptions (metrics.hpp:45-49) plus the number of ladder rungs
 * probed concurrently (the reference uses omp_get_max_threads(); 1 with a GPU). */
typedef struct {
    double qps_low;
    double max_qps;
    double rel_width;
    int32_t parallel;
} ssh_capacity_opts;

/* servesim::CapacityProbe (metrics.hpp:51-55) */
typedef struct {
    double qps;
    int32_t pass;
    ssh_latency report;
} ssh_capacity_probe;

/* Maximum sustainable qps under slo_ms (P99 TBT) with median scheduling delay
 * <= 2 s (meets_slo, metrics.cpp:65-67): every probe runs the reference
 * workload preset trace make_trace(workload, qps, probe_requests, seed) through
 * the engine with the cost model `params` — or, when sim->gpu is set, real
 * forwards on that context (then opts->parallel must be 1). SS_INFEASIBLE when
 * qps_low fails. probes (nullable) receives up to cap probes in search order. */
ss_status ssh_capacity_search(const ssh_replica_cfg* cfg, const ssh_cost_params* params,
                              const char* workload, int32_t probe_requests, uint64_t seed,
                              double slo_ms, const ssh_capacity_opts* opts, const ssh_sim_opts* sim,
                              double* qps_out, int32_t* monotone_warning,
                              ssh_capacity_probe* probes, int32_t cap, int32_t* n_probes);

int32_t ssh_next_chunk_size(int32_t prompt_tokens, int32_t prefill_done, int32_t token_budget,
                            int32_t packed_tokens, int32_t chunk_align);
ss_status ssh_percentile(const double* series, int64_t n, double p, double* out);

/* Host-built GPU descriptors for explicit batches (tests, benches). Each
 * entry gets its own request id (= its index); the ledger grows every entry to
 * prefix + tokens in entry order, exactly as Engine::try_issue does. A chunk
 * entry produces logits when completes[e] != 0 (NULL: every chunk completes). */
typedef struct ssh_desc ssh_desc;
ss_status ssh_desc_build(const ssh_entry* entries, int32_t n, const int32_t* completes,
                         int32_t block_size, int32_t vocab, uint64_t token_seed, ssh_desc** out);
/* Canonical hybrid batch of sched.cpp:159-169: n_dec decodes at kv_each cached
 * tokens plus one prompt-completing chunk of tau - n_dec tokens at chunk_prefix. */
ss_status ssh_desc_canonical(int32_t tau, int32_t n_dec, int64_t kv_each, int64_t chunk_prefix,
                             int32_t block_size, int32_t vocab, uint64_t token_seed, ssh_desc** out);
/* The descriptor view (pointers stay valid until ssh_desc_free). */
const ss_batch_desc* ssh_desc_view(const ssh_desc* d);
/* Blocks spanned by all tables (max id + 1): the KV pool size it needs. */
int64_t ssh_desc_pool_blocks(const ssh_desc* d);
void ssh_desc_free(ssh_desc* d);

/* Replay session: a persistent KV ledger + block tables for executing an
 * externally given micro-batch stream (e.g. the reference's golden batch
 * stream) on the GPU or the oracle. Each step grows every entry's request to
 * prefix + tokens in entry order (admitting requests on first sight), exactly
 * as Engine::try_issue does (engine.cpp:207-221); ssh_session_release returns
 * a finished request's blocks (engine.cpp:283-286). Token ids use the real
 * request ids. prompt_lens[e] marks chunk entries that complete their prompt. */
typedef struct ssh_session ssh_session;
ss_status ssh_session_create(int64_t kv_blocks, int32_t block_size, int32_t vocab, uint64_t token_seed,
                             ssh_session** out);
ss_status ssh_session_step(ssh_session* s, const ssh_entry* entries, int32_t n, const int32_t* prompt_lens,
                           ssh_desc** out);
ss_status ssh_session_release(ssh_session* s, int32_t request_id);
int64_t ssh_session_peak_blocks(const ssh_session* s);
void ssh_session_free(ssh_session* s);

const char* ssh_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* SS_HOST_H */
