#include "sched.hpp"

#include <algorithm>
#include <string>

namespace ss {

namespace {

bool is_ready(int rid, const InFlight& in_flight) { return in_flight.count(rid) == 0; }

bool fits(const KvLedger& kv, const Request& r, const ReplicaConfig& cfg) {
    return kv.can_admit(r.prompt, cfg.reserve_decode_tokens, cfg.watermark);
}

// Moves the head of the wait queue to running and commits its reservation.
void admit_head(SchedState& st, KvLedger& kv, const Request& r, const ReplicaConfig& cfg) {
    kv.admit(r.id, std::int64_t(r.prompt) + cfg.reserve_decode_tokens);
    st.waiting.pop_front();
    st.running.push_back(r.id);
}

void push_decodes(Batch& b, const SchedState& st, const std::vector<Request>& reqs, const InFlight& fl) {
    for (int id : st.running) {
        const Request& r = reqs[std::size_t(id)];
        if (r.phase == Phase::Decoding && is_ready(id, fl)) b.entries.push_back(decode_entry(r));
    }
}

bool running_full(const SchedState& st, int cap) { return int(st.running.size()) >= cap; }

}  // namespace

void SchedState::drop_running(int rid) {
    running.erase(std::remove(running.begin(), running.end(), rid), running.end());
}

int next_chunk(const Request& r, int budget, int packed, int align) {
    const int room = budget - packed;
    if (room <= 0) return 0;
    const int left = r.prefill_left();
    return left <= room ? left : (room / align) * align;
}

Batch stall_free_batch(SchedState& st, std::vector<Request>& reqs, KvLedger& kv,
                       const ReplicaConfig& cfg, const InFlight& fl) {
    Batch b;
    push_decodes(b, st, reqs, fl);  // (1) never stall a running decode
    int packed = int(b.entries.size());
    if (!cfg.hybrid_batching && packed > 0) return b;

    for (int id : st.running) {  // (2) continue in-progress prefills
        const Request& r = reqs[std::size_t(id)];
        if (r.prefill_complete() || !is_ready(id, fl)) continue;
        const int c = next_chunk(r, cfg.token_budget, packed, cfg.chunk_align);
        if (c > 0) {
            b.entries.push_back(chunk_entry(r, c));
            packed += c;
        }
    }
    while (!st.waiting.empty() && packed < cfg.token_budget) {  // (3) FCFS admissions
        const Request& r = reqs[std::size_t(st.waiting.front())];
        if (running_full(st, cfg.max_batch_size) || !fits(kv, r, cfg)) break;
        const int c = next_chunk(r, cfg.token_budget, packed, cfg.chunk_align);
        if (c == 0) break;
        admit_head(st, kv, r, cfg);
        b.entries.push_back(chunk_entry(r, c));
        packed += c;
    }
    return b;
}

Batch request_level_batch(SchedState& st, std::vector<Request>& reqs, KvLedger& kv,
                          const ReplicaConfig& cfg, const InFlight& fl) {
    Batch b;
    if (!st.running.empty()) {
        push_decodes(b, st, reqs, fl);
        return b;
    }
    while (!st.waiting.empty()) {
        const Request& r = reqs[std::size_t(st.waiting.front())];
        if (running_full(st, cfg.max_batch_size) || !fits(kv, r, cfg)) break;
        admit_head(st, kv, r, cfg);
        b.entries.push_back(chunk_entry(r, r.prompt));
    }
    return b;
}

Batch vllm_batch(SchedState& st, std::vector<Request>& reqs, KvLedger& kv,
                 const ReplicaConfig& cfg, const InFlight& fl) {
    Batch b;
    std::int64_t prompt_tokens = 0;
    while (!st.waiting.empty()) {
        const Request& r = reqs[std::size_t(st.waiting.front())];
        if (running_full(st, cfg.max_batch_size) || !fits(kv, r, cfg)) break;
        if (prompt_tokens + r.prompt > cfg.max_num_batched_tokens) {
            // The token cap yields to one oversized prompt, alone in its batch.
            if (b.entries.empty() && r.prompt > cfg.max_num_batched_tokens) {
                admit_head(st, kv, r, cfg);
                b.entries.push_back(chunk_entry(r, r.prompt));
            }
            break;
        }
        admit_head(st, kv, r, cfg);
        prompt_tokens += r.prompt;
        b.entries.push_back(chunk_entry(r, r.prompt));
    }
    if (b.empty()) push_decodes(b, st, reqs, fl);
    return b;
}

Batch orca_batch(SchedState& st, std::vector<Request>& reqs, KvLedger& kv,
                 const ReplicaConfig& cfg, const InFlight& fl) {
    Batch b;
    push_decodes(b, st, reqs, fl);
    while (!st.waiting.empty()) {
        const Request& r = reqs[std::size_t(st.waiting.front())];
        if (running_full(st, cfg.orca_cap()) || !fits(kv, r, cfg)) break;
        admit_head(st, kv, r, cfg);
        b.entries.push_back(chunk_entry(r, r.prompt));
    }
    return b;
}

Batch form_batch(SchedState& st, std::vector<Request>& reqs, KvLedger& kv,
                 const ReplicaConfig& cfg, const InFlight& fl) {
    switch (cfg.policy) {
        case Policy::RequestLevel: return request_level_batch(st, reqs, kv, cfg, fl);
        case Policy::Vllm: return vllm_batch(st, reqs, kv, cfg, fl);
        case Policy::Orca: return orca_batch(st, reqs, kv, cfg, fl);
        case Policy::StallFree: return stall_free_batch(st, reqs, kv, cfg, fl);
    }
    throw ContractViolation("unknown scheduler policy");
}

int token_budget_for(double t_max_ms, const CostParams& p, int pp, int rep_decodes,
                     std::int64_t rep_kv, int align, int max_budget, double factor_override) {
    const double factor = factor_override > 0.0 ? factor_override : double(pp);
    int best = 0;
    for (int tau = align; tau <= max_budget; tau += align) {
        if (tau - rep_decodes < 1) continue;
        if (iteration_time(canonical_batch(tau, rep_decodes, rep_kv, 0), p) * factor <= t_max_ms) best = tau;
    }
    if (best == 0)
        throw InfeasibleSlo("no token budget satisfies TBT target of " + std::to_string(t_max_ms) + " ms");
    return best;
}

}  // namespace ss
