// Paged KV ledger + block tables.
//
// The counting semantics restate KvCacheState (reference
// proj/include/servesim/kvcache.hpp:22-65, proj/src/kvcache.cpp:8-62): physical
// blocks follow resident tokens, a commitment ledger follows admission-time
// reservations, admission holds back a watermark. The reference tracks counts
// only; the GPU needs physical block ids, so this ledger also owns a
// deterministic allocator: a LIFO free list whose initial order hands out ids
// 0, 1, 2, ... and which reuses the most recently freed id first. Block ids
// are assigned in grow() call order (entry order inside Engine::try_issue,
// engine.cpp:211-216), so table sizes equal allocated_for() at every step and
// the largest id ever issued is (peak concurrent blocks - 1).
#pragma once

#include <cstdint>
#include <vector>

#include "types.hpp"

namespace ss {

std::int64_t blocks_for(std::int64_t tokens, std::int64_t block_size);  // kvcache.cpp:8-12

class KvLedger {
public:
    KvLedger(std::int64_t total_blocks, std::int64_t block_size);

    bool can_admit(std::int64_t prompt, std::int64_t reserve, double watermark = 0.0) const;
    void admit(int rid, std::int64_t expected_tokens);
    void grow(int rid, std::int64_t new_tokens);
    void release(int rid);

    std::int64_t total() const { return total_; }
    std::int64_t block_size() const { return bs_; }
    std::int64_t free_blocks() const { return total_ - allocated_; }
    std::int64_t allocated() const { return allocated_; }
    std::int64_t committed() const { return committed_; }
    std::int64_t allocated_for(int rid) const;
    bool live(int rid) const;
    std::int64_t peak_allocated() const { return peak_; }

    // Physical block ids of a live request, in logical order.
    const std::vector<std::int32_t>& table(int rid) const;

private:
    struct Slot {
        bool live = false;
        std::int64_t tokens = 0;
        std::int64_t blocks = 0;
        std::int64_t committed = 0;
        std::vector<std::int32_t> ids;
    };
    Slot& at(int rid);
    const Slot* find(int rid) const;
    std::int32_t pop_id();

    std::int64_t total_;
    std::int64_t bs_;
    std::int64_t allocated_ = 0;
    std::int64_t committed_ = 0;
    std::int64_t peak_ = 0;
    std::vector<Slot> slots_;
    std::vector<std::int32_t> recycled_;  // LIFO of freed ids
    std::int64_t next_fresh_ = 0;         // ids never handed out start here
};

}  // namespace ss
