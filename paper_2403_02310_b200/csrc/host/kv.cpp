#include "kv.hpp"

#include <cmath>
#include <string>

namespace ss {

std::int64_t blocks_for(std::int64_t tokens, std::int64_t block_size) {
    if (tokens < 0 || block_size < 1) throw ContractViolation("invalid blocks_needed arguments");
    return tokens == 0 ? 0 : (tokens + block_size - 1) / block_size;
}

KvLedger::KvLedger(std::int64_t total_blocks, std::int64_t block_size)
    : total_(total_blocks), bs_(block_size) {
    if (total_blocks < 0 || block_size < 1) throw ContractViolation("invalid kv cache geometry");
}

bool KvLedger::can_admit(std::int64_t prompt, std::int64_t reserve, double watermark) const {
    const std::int64_t need = blocks_for(prompt + reserve, bs_);
    const auto held_back = static_cast<std::int64_t>(std::floor(watermark * double(total_)));
    return total_ - committed_ - held_back >= need;
}

KvLedger::Slot& KvLedger::at(int rid) {
    if (rid < 0) throw ContractViolation("negative request id");
    if (std::size_t(rid) >= slots_.size()) slots_.resize(std::size_t(rid) + 1);
    return slots_[std::size_t(rid)];
}

const KvLedger::Slot* KvLedger::find(int rid) const {
    if (rid < 0 || std::size_t(rid) >= slots_.size() || !slots_[std::size_t(rid)].live) return nullptr;
    return &slots_[std::size_t(rid)];
}

bool KvLedger::live(int rid) const { return find(rid) != nullptr; }

std::int64_t KvLedger::allocated_for(int rid) const {
    const Slot* s = find(rid);
    return s ? s->blocks : 0;
}

const std::vector<std::int32_t>& KvLedger::table(int rid) const {
    const Slot* s = find(rid);
    if (!s) throw ContractViolation("block table of a request that is not live");
    return s->ids;
}

void KvLedger::admit(int rid, std::int64_t expected_tokens) {
    Slot& s = at(rid);
    if (s.live) throw ContractViolation("request already live in kv cache");
    s = Slot{};
    s.live = true;
    s.committed = blocks_for(expected_tokens, bs_);
    committed_ += s.committed;
}

std::int32_t KvLedger::pop_id() {
    if (!recycled_.empty()) {
        const std::int32_t id = recycled_.back();
        recycled_.pop_back();
        return id;
    }
    return static_cast<std::int32_t>(next_fresh_++);
}

void KvLedger::grow(int rid, std::int64_t new_tokens) {
    Slot* s = const_cast<Slot*>(find(rid));
    if (!s) throw ContractViolation("grow on unknown request");
    if (new_tokens < s->tokens) throw ContractViolation("kv allocation cannot shrink");
    const std::int64_t want = blocks_for(new_tokens, bs_);
    const std::int64_t delta = want - s->blocks;
    if (delta > free_blocks())
        throw OutOfKvBlocks("out of KV blocks while growing request " + std::to_string(rid));
    for (std::int64_t i = 0; i < delta; ++i) s->ids.push_back(pop_id());
    allocated_ += delta;
    if (allocated_ > peak_) peak_ = allocated_;
    if (want > s->committed) {
        committed_ += want - s->committed;
        s->committed = want;
    }
    s->blocks = want;
    s->tokens = new_tokens;
}

void KvLedger::release(int rid) {
    Slot* s = const_cast<Slot*>(find(rid));
    if (!s) throw ContractViolation("release on unknown request");
    allocated_ -= s->blocks;
    committed_ -= s->committed;
    for (std::int32_t id : s->ids) recycled_.push_back(id);
    *s = Slot{};
}

}  // namespace ss
