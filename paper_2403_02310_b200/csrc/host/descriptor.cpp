#include "descriptor.hpp"

#include <algorithm>

#include "../../../include/ss_synth.h"

namespace ss {

ss_batch_desc HostDesc::view() const {
    ss_batch_desc d{};
    d.num_entries = std::int32_t(ctx_len.size());
    d.num_tokens = std::int32_t(pos.size());
    d.cu_q = cu_q.data();
    d.ctx_len = ctx_len.data();
    d.pos = pos.data();
    d.token_ids = token_ids.data();
    d.slot = slot.data();
    d.block_table = block_table.data();
    d.max_blocks = max_blocks;
    d.out_rows = out_rows.data();
    d.n_out = std::int32_t(out_rows.size());
    return d;
}

HostDesc build_desc(const Batch& b, const KvLedger& kv, const std::vector<bool>& completes,
                    std::uint64_t token_seed, std::int32_t vocab) {
    HostDesc d;
    const std::int64_t bs = kv.block_size();
    const std::size_t E = b.entries.size();
    std::int32_t maxb = 1;
    for (const Entry& e : b.entries) maxb = std::max<std::int32_t>(maxb, std::int32_t(kv.table(e.rid).size()));
    d.max_blocks = maxb;
    d.block_table.assign(E * std::size_t(maxb), -1);
    d.cu_q.push_back(0);
    for (std::size_t i = 0; i < E; ++i) {
        const Entry& e = b.entries[i];
        const auto& tbl = kv.table(e.rid);
        const std::int64_t ctx = e.prefix + e.tokens;
        if (blocks_for(ctx, bs) > std::int64_t(tbl.size()))
            throw ContractViolation("block table does not cover the entry's positions");
        std::copy(tbl.begin(), tbl.end(), d.block_table.begin() + std::ptrdiff_t(i * std::size_t(maxb)));
        d.rids.push_back(e.rid);
        d.ctx_len.push_back(std::int32_t(ctx));
        for (int j = 0; j < e.tokens; ++j) {
            const std::int64_t p = e.prefix + j;
            d.pos.push_back(std::int32_t(p));
            d.token_ids.push_back(ss_token_id(token_seed, e.rid, p, vocab));
            d.slot.push_back(std::int64_t(tbl[std::size_t(p / bs)]) * bs + p % bs);
        }
        d.cu_q.push_back(std::int32_t(d.pos.size()));
        if (e.kind == Kind::Decode || completes[i]) d.out_rows.push_back(std::int32_t(d.pos.size()) - 1);
    }
    return d;
}

HostDesc build_desc(const Batch& b, const KvLedger& kv, const std::vector<Request>& reqs,
                    std::uint64_t token_seed, std::int32_t vocab) {
    std::vector<bool> completes;
    for (const Entry& e : b.entries)
        completes.push_back(e.kind == Kind::Decode ||
                            e.prefix + e.tokens == std::int64_t(reqs[std::size_t(e.rid)].prompt));
    return build_desc(b, kv, completes, token_seed, vocab);
}

}  // namespace ss
