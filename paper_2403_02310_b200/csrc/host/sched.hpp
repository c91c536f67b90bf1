// Batch formation: the stall-free policy (the hot path) and the three baseline
// policies it is compared against. Restates reference proj/src/sched.cpp.
//
// Entry order in the returned Batch is the packed token order the GPU forward
// consumes: ready decodes first (running order), then in-progress chunks, then
// FCFS admissions (sched.cpp:105-137).
#pragma once

#include <deque>
#include <unordered_set>
#include <vector>

#include "costmodel.hpp"
#include "kv.hpp"
#include "types.hpp"

namespace ss {

struct SchedState {  // sched.hpp:16-21
    std::deque<int> waiting;  // FCFS
    std::vector<int> running; // admission order
    void drop_running(int rid);
};

using InFlight = std::unordered_set<int>;  // ids whose last entry has not exited

// get_next_chunk_size, sched.cpp:97-103: the final chunk passes unaligned,
// others are floored to chunk_align; 0 when no aligned room is left.
int next_chunk(const Request& r, int budget, int packed, int align);

Batch stall_free_batch(SchedState& st, std::vector<Request>& reqs, KvLedger& kv,
                       const ReplicaConfig& cfg, const InFlight& in_flight);
Batch request_level_batch(SchedState& st, std::vector<Request>& reqs, KvLedger& kv,
                          const ReplicaConfig& cfg, const InFlight& in_flight);
Batch vllm_batch(SchedState& st, std::vector<Request>& reqs, KvLedger& kv,
                 const ReplicaConfig& cfg, const InFlight& in_flight);
Batch orca_batch(SchedState& st, std::vector<Request>& reqs, KvLedger& kv,
                 const ReplicaConfig& cfg, const InFlight& in_flight);
Batch form_batch(SchedState& st, std::vector<Request>& reqs, KvLedger& kv,
                 const ReplicaConfig& cfg, const InFlight& in_flight);

// compute_token_budget, sched.cpp:154-175 (one-time profiling over tau).
int token_budget_for(double t_max_ms, const CostParams& p, int pp, int rep_decodes = 32,
                     std::int64_t rep_kv = 4096, int align = 32, int max_budget = 8192,
                     double factor_override = 0.0);

}  // namespace ss
