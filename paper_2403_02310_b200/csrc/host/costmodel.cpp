#include "costmodel.hpp"

#include <algorithm>

namespace ss {

void CostParams::validate() const {
    if (per_token_linear_ms < 0 || attn_prefill_quad_ms < 0 || attn_kv_read_ms < 0 ||
        attn_decode_per_kv_ms < 0 || fixed_overhead_ms < 0 || tp_comm_ms < 0 || pp_send_ms < 0)
        throw ContractViolation("timing constants must be non-negative");
    if (saturation_tokens < 1) throw ContractViolation("saturation_tokens must be >= 1");
    if (tile_size < 1) throw ContractViolation("tile_size must be >= 1");
    if (tile_penalty_frac < 0) throw ContractViolation("tile_penalty_frac must be >= 0");
}

double iteration_time(const Batch& b, const CostParams& p, int tp, int pp) {
    if (b.empty()) return 0.0;
    const std::int64_t t = b.tokens();
    // Linear operators: roofline floor vs per-token slope, the slope paying the
    // tile-quantisation penalty off multiples of tile_size.
    const double pen = (t <= 0 || p.tile_size <= 1 || t % p.tile_size == 0) ? 1.0 : 1.0 + p.tile_penalty_frac;
    const double linear = std::max(p.mem_floor_ms(), p.per_token_linear_ms * double(t) * pen) / double(tp);
    double attn = 0.0;
    for (const Entry& e : b.entries) {
        if (e.kind == Kind::Chunk) {
            const double c = double(e.tokens);
            attn += p.attn_prefill_quad_ms * c * c + p.attn_kv_read_ms * c * double(e.prefix);
        } else {
            attn += p.attn_decode_per_kv_ms * double(e.prefix);
        }
    }
    return (p.fixed_overhead_ms + linear + attn + p.tp_comm_ms) / double(pp);
}

Batch decode_batch(int n, std::int64_t kv_each) {
    Batch b;
    for (int i = 0; i < n; ++i) b.entries.push_back(Entry{i, Kind::Decode, 1, kv_each});
    return b;
}

Batch prefill_batch(std::int64_t prompt) {
    Batch b;
    b.entries.push_back(Entry{0, Kind::Chunk, int(prompt), 0});
    return b;
}

double decode_reference_time(const CostParams& p) { return iteration_time(decode_batch(32, 4096), p); }

Batch canonical_batch(int tau, int n_dec, std::int64_t kv_each, std::int64_t chunk_prefix) {
    Batch b = decode_batch(n_dec, kv_each);
    b.entries.push_back(Entry{n_dec, Kind::Chunk, tau - n_dec, chunk_prefix});
    return b;
}

std::optional<CostParams> cost_preset(const std::string& name) {
    CostParams p;
    if (name == "mistral7b") {
        p.per_token_linear_ms = 0.0263671875;
        p.saturation_tokens = 512;
        p.attn_prefill_quad_ms = 2.0e-7;
        p.attn_kv_read_ms = 4.2e-7;
        p.attn_decode_per_kv_ms = 3.4332275390625e-05;
        p.fixed_overhead_ms = 2.0;
        p.pp_send_ms = 1.0;
    } else if (name == "yi34b") {
        p.per_token_linear_ms = 0.33;
        p.saturation_tokens = 43;
        p.attn_prefill_quad_ms = 3.0e-7;
        p.attn_kv_read_ms = 6.3e-7;
        p.attn_decode_per_kv_ms = 6.1798095703125e-06;
        p.fixed_overhead_ms = 25.0;
        p.pp_send_ms = 1.0;
    } else if (name == "llama70b") {
        p.per_token_linear_ms = 1.5;
        p.saturation_tokens = 100;
        p.attn_prefill_quad_ms = 7.0e-7;
        p.attn_kv_read_ms = 1.47e-6;
        p.attn_decode_per_kv_ms = 3.509521484375e-04;
        p.fixed_overhead_ms = 4.0;
        p.pp_send_ms = 3.0;
    } else if (name == "falcon180b") {
        p.per_token_linear_ms = 0.244140625;
        p.saturation_tokens = 512;
        p.attn_prefill_quad_ms = 8.6e-6;
        p.attn_kv_read_ms = 1.806e-5;
        p.attn_decode_per_kv_ms = 5.340576171875e-04;
        p.fixed_overhead_ms = 5.0;
        p.pp_send_ms = 2.0;
    } else if (name == "tiny") {
        p.fixed_overhead_ms = 1.0;
        p.per_token_linear_ms = 0.01;
        p.saturation_tokens = 100;
        p.attn_prefill_quad_ms = 1e-6;
        p.attn_kv_read_ms = 2e-6;
        p.attn_decode_per_kv_ms = 1e-5;
        p.pp_send_ms = 0.0;
    } else {
        return std::nullopt;
    }
    return p;
}

}  // namespace ss
