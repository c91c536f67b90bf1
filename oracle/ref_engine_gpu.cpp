// TEST INFRASTRUCTURE ONLY. The reference's OWN engine driving the B200 forward: the build
// (oracle/Makefile, target ref_engine_gpu) compiles the reference's src/engine.cpp with exactly
// one line changed — the model step at engine.cpp:227,
//     const double iter_ms = iteration_time(batch, params_, cfg_.tp_degree, cfg_.pp_degree);
// becomes
//     const double iter_ms = g_gpu_step ? g_gpu_step(batch) : iteration_time(...);
// (sed at build time; no reference source is stored in this repo) — and links it with the
// reference's other sources and this driver. This is the INTEGRATION.md §2 patch, compiled
// against the reference itself. The reference ledger counts blocks only, so the step builds
// each batch's descriptor with fresh block tables (ssh_desc_build): the forward reads and
// writes the same number of K/V pages as with persistent tables, so the measured time — all
// the reference's model step returns — is the same work.
//
//   ref_engine_gpu <layers> <hidden> <q_heads> <kv_heads> <head_dim> <ffn> <vocab> <rope_theta>
//                  <preset> <workload> <qps> <n_requests> <seed> <token_budget> <kv_pool_blocks>
// prints one JSON line: the reference's summarize() of its own simulate() run.
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "servesim/costmodel.hpp"
#include "servesim/engine.hpp"
#include "servesim/metrics.hpp"
#include "servesim/presets.hpp"
#include "servesim/workload.hpp"
#include "ss_gpu.h"
#include "ss_host.h"

namespace servesim {
double (*g_gpu_step)(const Batch&) = nullptr;  // the engine.cpp:227 hook (declared by the sed patch)
}

namespace {
ss_ctx* g_ctx = nullptr;
int g_vocab = 0;
long g_steps = 0;
double g_step_ms = 0.0;

double gpu_step(const servesim::Batch& b) {
    std::vector<ssh_entry> e;
    e.reserve(b.entries.size());
    for (const auto& x : b.entries)
        e.push_back(ssh_entry{x.request_id, x.kind == servesim::EntryKind::PrefillChunk ? 1 : 0, x.chunk_tokens,
                              x.prefix_tokens});
    ssh_desc* d = nullptr;
    if (ssh_desc_build(e.data(), int32_t(e.size()), nullptr, 16, g_vocab, 7, &d) != SS_OK)
        throw std::runtime_error("ssh_desc_build failed");
    float ms = 0.f;
    const ss_status st = ss_forward_hybrid(g_ctx, ssh_desc_view(d), nullptr, nullptr, &ms);
    ssh_desc_free(d);
    if (st != SS_OK) throw std::runtime_error(std::string("ss_forward_hybrid: ") + ss_last_error(g_ctx));
    ++g_steps;
    g_step_ms += ms;
    return double(ms);
}
}  // namespace

int main(int argc, char** argv) {
    if (argc != 16) {
        std::fprintf(stderr, "usage: %s layers hidden q_heads kv_heads head_dim ffn vocab rope_theta preset workload "
                             "qps n seed token_budget kv_pool_blocks\n", argv[0]);
        return 2;
    }
    ss_model_cfg mc{};
    mc.num_layers = std::atoi(argv[1]);
    mc.hidden = std::atoi(argv[2]);
    mc.num_q_heads = std::atoi(argv[3]);
    mc.num_kv_heads = std::atoi(argv[4]);
    mc.head_dim = std::atoi(argv[5]);
    mc.ffn = std::atoi(argv[6]);
    mc.vocab = std::atoi(argv[7]);
    mc.rope_theta = float(std::atof(argv[8]));
    mc.rms_eps = 1e-5f;
    mc.max_positions = 16384 + 1024;
    g_vocab = mc.vocab;
    if (ss_create(&mc, 0, 1, nullptr, 1234, 0, &g_ctx) != SS_OK) {
        std::fprintf(stderr, "ss_create: %s\n", ss_last_error(nullptr));
        return 1;
    }
    const long pool = std::atol(argv[15]);
    if (ss_kv_alloc(g_ctx, pool, 16) != SS_OK) {
        std::fprintf(stderr, "ss_kv_alloc: %s\n", ss_last_error(g_ctx));
        return 1;
    }
    const auto params = servesim::model_preset(argv[9]);
    const auto wl = servesim::workload_preset(argv[10]);
    if (!params || !wl) {
        std::fprintf(stderr, "unknown preset / workload\n");
        return 2;
    }
    servesim::ReplicaConfig cfg;
    cfg.token_budget = std::atoi(argv[14]);
    cfg.kv_blocks = pool;
    const auto trace = servesim::make_trace(*wl, std::atof(argv[11]), std::atoi(argv[12]), std::strtoull(argv[13], nullptr, 10));
    servesim::SimOptions so;
    so.keep_events = false;
    servesim::g_gpu_step = gpu_step;
    const servesim::SimReport rep = servesim::simulate(cfg, *params, trace, so);
    const servesim::LatencyReport s = servesim::summarize(rep);
    std::printf("{\"tbt_p99_ms\": %.4f, \"tbt_median_ms\": %.4f, \"ttft_median_ms\": %.4f, \"throughput_tps\": %.3f, "
                "\"n_requests\": %d, \"microbatches\": %lld, \"gpu_steps\": %ld, \"mean_step_ms\": %.4f}\n",
                s.tbt_p99_ms, s.tbt_median_ms, s.ttft_median_ms, s.throughput_tps, s.n_requests,
                (long long)rep.num_microbatches, g_steps, g_steps ? g_step_ms / double(g_steps) : 0.0);
    ss_destroy(g_ctx);
    return 0;
}
