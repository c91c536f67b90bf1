// The reference's analytical model step and its presets.
//
// iteration_time() is the CPU "model step" the GPU forward replaces (reference
// proj/src/costmodel.cpp:39-56). It stays here for three reasons: the engine's
// CostModelExecutor must reproduce the reference's clock bit for bit (golden
// event logs), compute_token_budget's one-time profiling still uses it, and the
// SLO thresholds are derived from decode_reference_time (metrics.cpp:61-64).
#pragma once

#include <optional>
#include <string>
#include <vector>

#include "types.hpp"

namespace ss {

struct CostParams {  // costmodel.hpp:19-41
    double per_token_linear_ms = 0.0;
    int saturation_tokens = 1;
    double attn_prefill_quad_ms = 0.0;
    double attn_kv_read_ms = 0.0;
    double attn_decode_per_kv_ms = 0.0;
    double fixed_overhead_ms = 0.0;
    double tp_comm_ms = 0.0;
    double pp_send_ms = 0.0;
    int tile_size = 256;
    double tile_penalty_frac = 0.32;

    double mem_floor_ms() const { return per_token_linear_ms * saturation_tokens; }
    void validate() const;
};

double iteration_time(const Batch& b, const CostParams& p, int tp = 1, int pp = 1);
Batch decode_batch(int n, std::int64_t kv_each);   // make_decode_batch, costmodel.cpp:58-70
Batch prefill_batch(std::int64_t prompt);          // make_prefill_batch, costmodel.cpp:72-81
double decode_reference_time(const CostParams& p); // 32 decodes at 4k KV

// presets.cpp:8-66, plus the unit-test clock of test_engine.cpp:14-25 ("tiny").
std::optional<CostParams> cost_preset(const std::string& name);

// Canonical hybrid batch of sched.cpp:159-169: n_dec decodes at kv_each plus
// one chunk of (tau - n_dec) tokens at `chunk_prefix`.
Batch canonical_batch(int tau, int n_dec = 32, std::int64_t kv_each = 4096, std::int64_t chunk_prefix = 0);

}  // namespace ss
