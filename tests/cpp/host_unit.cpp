// C++ unit tests of the host restatement's internals (scheduler states, KV
// ledger + block allocator), mirroring the reference's doctest cases
// (reference proj/tests/test_sched.cpp, test_kvcache.cpp, test_core.cpp).
// Built and run by tests/test_host_unit.py.
#include <cstdio>
#include <functional>
#include <random>
#include <set>
#include <string>
#include <unordered_map>
#include <vector>

#include "engine.hpp"
#include "kv.hpp"
#include "sched.hpp"

using namespace ss;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                             \
    do {                                                                     \
        ++g_checks;                                                          \
        if (!(c)) {                                                          \
            ++g_fail;                                                        \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);         \
        }                                                                    \
    } while (0)
#define CHECK_THROWS(expr, T)                                                \
    do {                                                                     \
        bool thrown = false;                                                 \
        try { expr; } catch (const T&) { thrown = true; }                    \
        CHECK(thrown);                                                       \
    } while (0)

struct World {  // test_sched.cpp:12-57
    std::vector<Request> reqs;
    SchedState st;
    KvLedger kv{1 << 20, 16};
    ReplicaConfig cfg;
    InFlight fl;
    World() { cfg.kv_blocks = 1 << 20; cfg.watermark = 0.0; }
    int queued(int p, int o) { int id = int(reqs.size()); reqs.emplace_back(id, 0, p, o); st.waiting.push_back(id); return id; }
    int decoding(int p, int o, int done = 1) {
        int id = int(reqs.size()); Request r(id, 0, p, o); r.prefill_done = p; r.decodes_done = done; r.phase = Phase::Decoding;
        reqs.push_back(r); st.running.push_back(id); kv.admit(id, p); kv.grow(id, p + done - 1); return id;
    }
    int mid_prefill(int p, int o, int done) {
        int id = int(reqs.size()); Request r(id, 0, p, o); r.prefill_done = done; r.phase = Phase::Prefilling;
        reqs.push_back(r); st.running.push_back(id); kv.admit(id, p); kv.grow(id, done); return id;
    }
    Batch next() { return form_batch(st, reqs, kv, cfg, fl); }
};

static int count(const Batch& b, Kind k) { int n = 0; for (auto& e : b.entries) n += e.kind == k; return n; }

static void sched_tests() {
    { World w; w.cfg.policy = Policy::RequestLevel; w.decoding(100, 5); w.decoding(200, 5); w.queued(500, 5);
      Batch b = w.next(); CHECK(b.entries.size() == 2); CHECK(count(b, Kind::Decode) == 2); CHECK(w.st.waiting.size() == 1); }
    { World w; w.cfg.policy = Policy::RequestLevel; w.queued(500, 5); w.queued(700, 5); Batch b = w.next();
      CHECK(b.entries.size() == 2 && b.entries[0].tokens == 500 && b.entries[1].tokens == 700); CHECK(w.st.running.size() == 2); }
    { World w; w.cfg.policy = Policy::Vllm; w.decoding(100, 5); w.decoding(200, 5); int c = w.queued(900, 5); Batch b = w.next();
      CHECK(b.entries.size() == 1 && b.entries[0].rid == c && b.entries[0].tokens == 900); }
    { World w; w.cfg.policy = Policy::Vllm; w.queued(1730, 5); w.queued(1730, 5); w.queued(1730, 5); Batch b = w.next();
      CHECK(b.entries.size() == 2 && b.prefill_tokens() == 3460 && w.st.waiting.size() == 1); }
    { World w; w.cfg.policy = Policy::Vllm; w.decoding(100, 5); int c = w.queued(9000, 5); int d = w.queued(100, 5); Batch b = w.next();
      CHECK(b.entries.size() == 1 && b.entries[0].rid == c && b.entries[0].tokens == 9000 && w.st.waiting.front() == d); }
    { World w; w.cfg.policy = Policy::Orca; w.decoding(100, 5); w.decoding(200, 5); int c = w.queued(700, 5); Batch b = w.next();
      CHECK(b.entries.size() == 3 && count(b, Kind::Decode) == 2 && b.entries[2].rid == c && b.entries[2].tokens == 700); }
    { World w; w.cfg.policy = Policy::Orca; w.cfg.max_batch_size = 8; CHECK(w.cfg.orca_cap() == 2);
      w.decoding(100, 50); w.decoding(100, 50); w.queued(300, 5); CHECK(count(w.next(), Kind::Chunk) == 0); }
    { World w; w.cfg.token_budget = 512; int a = w.decoding(100, 5); int b_ = w.decoding(200, 5); int c = w.mid_prefill(1000, 5, 300);
      Batch b = w.next(); CHECK(b.entries.size() == 3 && b.entries[0].rid == a && b.entries[1].rid == b_ && b.entries[2].rid == c);
      CHECK(b.entries[2].kind == Kind::Chunk && b.entries[2].tokens == 480 && b.tokens() == 482); }
    { World w; w.decoding(100, 5); w.decoding(200, 5); Batch b = w.next(); CHECK(b.prefill_tokens() == 0 && b.tokens() == 2); }
    { World w; w.cfg.token_budget = 2048; int c = w.queued(4096, 5); Batch b = w.next();
      CHECK(b.entries.size() == 1 && b.entries[0].rid == c && b.entries[0].tokens == 2048 && w.reqs[std::size_t(c)].phase == Phase::Queued); }
    { World w; w.cfg.token_budget = 512; w.queued(200, 5); w.queued(200, 5); w.queued(200, 5); Batch b = w.next();
      CHECK(b.entries.size() == 3 && b.entries[2].tokens == 96 && b.tokens() == 496); }
    { World w; w.cfg.hybrid_batching = false; w.decoding(100, 5); w.queued(400, 5); Batch b = w.next();
      CHECK(b.prefill_tokens() == 0); w.fl.insert(w.st.running[0]); Batch b2 = w.next();
      CHECK(count(b2, Kind::Decode) == 0 && b2.prefill_tokens() == 400); }
    for (Policy pol : {Policy::RequestLevel, Policy::Vllm, Policy::Orca, Policy::StallFree}) {
        World w; w.cfg.policy = pol; w.cfg.token_budget = 4096;
        int a = w.queued(100, 2), b_ = w.queued(100, 2), c = w.queued(100, 2); Batch b = w.next();
        std::vector<int> order; for (auto& e : b.entries) if (e.kind == Kind::Chunk) order.push_back(e.rid);
        CHECK((order == std::vector<int>{a, b_, c}));
    }
}

static void kv_tests() {
    CHECK(blocks_for(0, 16) == 0); CHECK(blocks_for(100, 16) == 7); CHECK(blocks_for(128, 16) == 8);
    CHECK_THROWS(blocks_for(-1, 16), ContractViolation);
    { KvLedger kv(10, 16); CHECK(kv.can_admit(100, 0)); KvLedger s(6, 16); CHECK(!s.can_admit(100, 0));
      KvLedger t(7, 16); CHECK(!t.can_admit(100, 16)); CHECK(t.can_admit(100, 0)); }
    { KvLedger kv(100, 16); CHECK(kv.can_admit(16 * 90, 0, 0.0)); CHECK(!kv.can_admit(16 * 91, 0, 0.10)); CHECK(kv.can_admit(16 * 90, 0, 0.10)); }
    { KvLedger kv(100, 16); kv.admit(1, 100); kv.grow(1, 100); CHECK(kv.allocated_for(1) == 7);
      auto f = kv.free_blocks(); kv.grow(1, 112); CHECK(kv.allocated_for(1) == 7 && kv.free_blocks() == f);
      kv.grow(1, 113); CHECK(kv.allocated_for(1) == 8 && kv.free_blocks() == f - 1);
      CHECK_THROWS(kv.grow(1, 100), ContractViolation);
      CHECK(kv.table(1).size() == 8); for (int i = 0; i < 8; ++i) CHECK(kv.table(1)[std::size_t(i)] == i); }
    { KvLedger kv(2, 16); kv.admit(1, 32); kv.grow(1, 32); CHECK(kv.free_blocks() == 0); CHECK_THROWS(kv.grow(1, 33), OutOfKvBlocks); }
    { KvLedger kv(100, 16); kv.admit(1, 128); kv.grow(1, 128); auto f = kv.free_blocks(); kv.release(1);
      CHECK(kv.free_blocks() == f + 8 && kv.allocated_for(1) == 0 && !kv.live(1)); CHECK_THROWS(kv.release(1), ContractViolation); }
    // Conservation + block-id invariants over random op sequences (test_kvcache.cpp:71-114):
    // tables are disjoint, sized like the ledger, and ids stay below the peak.
    std::mt19937_64 gen(1234);
    for (int round = 0; round < 50; ++round) {
        const std::int64_t total = 64 + std::int64_t(gen() % 512);
        KvLedger kv(total, 16);
        std::unordered_map<int, std::int64_t> ledger;
        int next = 0;
        for (int step = 0; step < 300; ++step) {
            const int op = int(gen() % 3);
            if (op == 0) {
                const std::int64_t tok = 1 + std::int64_t(gen() % 600);
                if (kv.can_admit(tok, 0)) { kv.admit(next, tok); kv.grow(next, tok); ledger[next] = tok; ++next; }
            } else if (op == 1 && !ledger.empty()) {
                auto it = ledger.begin(); std::advance(it, long(gen() % ledger.size()));
                const std::int64_t want = it->second + 1 + std::int64_t(gen() % 32);
                if (blocks_for(want, 16) - blocks_for(it->second, 16) <= kv.free_blocks()) { kv.grow(it->first, want); it->second = want; }
            } else if (!ledger.empty()) {
                auto it = ledger.begin(); std::advance(it, long(gen() % ledger.size())); kv.release(it->first); ledger.erase(it);
            }
            std::int64_t expect = 0; std::set<int> ids;
            for (auto& [id, tok] : ledger) {
                expect += blocks_for(tok, 16);
                CHECK(kv.allocated_for(id) == blocks_for(tok, 16));
                CHECK(std::int64_t(kv.table(id).size()) == blocks_for(tok, 16));
                for (int b : kv.table(id)) { CHECK(b >= 0 && b < kv.peak_allocated()); CHECK(ids.insert(b).second); }
            }
            CHECK(kv.allocated() == expect && kv.free_blocks() + kv.allocated() == total);
            CHECK(kv.peak_allocated() <= total);
        }
    }
}

static void core_tests() {
    Request r(0, 0, 100, 3);
    CHECK_THROWS(decode_entry(r), ContractViolation);
    Entry c = chunk_entry(r, 60); apply_result(r, c, 10); CHECK(r.phase == Phase::Prefilling && r.prefill_done == 60);
    CHECK_THROWS(chunk_entry(r, 41), ContractViolation);
    apply_result(r, chunk_entry(r, 40), 20); CHECK(r.phase == Phase::Decoding && r.first_token && *r.first_token == 20 && r.decodes_done == 1);
    Entry d = decode_entry(r); CHECK(d.prefix == 100);
    CHECK_THROWS(apply_result(r, d, 20), ContractViolation);  // emission times strictly increase
    apply_result(r, d, 30); apply_result(r, decode_entry(r), 40); CHECK(r.finished() && r.emits.size() == 3);
}

int main() {
    sched_tests();
    kv_tests();
    core_tests();
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
