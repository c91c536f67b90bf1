// Batch -> GPU descriptor (the arrays of ss_batch_desc, include/ss_gpu.h).
//
// Positions follow the reference's entry semantics (core.cpp:42-63,
// engine.cpp:211-216): a decode entry processes the token at position `prefix`
// and leaves prefix+1 tokens cached; a chunk processes [prefix, prefix+tokens).
// slot = table[pos / bs] * bs + pos % bs over the ledger's block tables.
#pragma once

#include <cstdint>
#include <vector>

#include "../../../include/ss_gpu.h"
#include "kv.hpp"
#include "types.hpp"

namespace ss {

struct HostDesc {
    std::vector<std::int32_t> cu_q, ctx_len, pos, token_ids, block_table, out_rows, rids;
    std::vector<std::int64_t> slot;
    std::int32_t max_blocks = 0;
    ss_batch_desc view() const;
};

// `completes[e]` says whether entry e produces logits: always for decodes;
// for chunks when prefix + tokens equals the request's prompt length.
HostDesc build_desc(const Batch& b, const KvLedger& kv, const std::vector<bool>& completes,
                    std::uint64_t token_seed, std::int32_t vocab);

// For engine batches: completion follows the live request state.
HostDesc build_desc(const Batch& b, const KvLedger& kv, const std::vector<Request>& reqs,
                    std::uint64_t token_seed, std::int32_t vocab);

}  // namespace ss
