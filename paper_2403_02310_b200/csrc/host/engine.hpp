// Discrete-event serving engine with a pluggable model step.
//
// Restates the reference engine (proj/src/engine.cpp:132-291): an event heap
// ordered (time, exit < first-stage-free < arrival, seq); each issue forms a
// batch, grows KV in entry order, asks the model step for the iteration time,
// converts it with max(1, llround(ms*1000)) and schedules the exit. The one
// structural change is the StepExecutor seam at the model step
// (engine.cpp:227): CostModelExecutor reproduces the reference clock bit for
// bit; the GPU executor (gpu_executor.cpp) runs the real hybrid-batch forward
// through the ss_gpu.h C ABI and returns the measured device time.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "costmodel.hpp"
#include "kv.hpp"
#include "sched.hpp"
#include "types.hpp"

namespace ss {

struct StepExecutor {
    virtual ~StepExecutor() = default;
    // Called once per issued batch, after the batch's KV growth, so the ledger's
    // block tables already cover every position the batch writes.
    virtual double step_ms(const Batch& b, const KvLedger& kv, const std::vector<Request>& reqs) = 0;
};

class CostModelExecutor final : public StepExecutor {
public:
    CostModelExecutor(CostParams p, int tp, int pp) : p_(p), tp_(tp), pp_(pp) {}
    double step_ms(const Batch& b, const KvLedger&, const std::vector<Request>&) override {
        return iteration_time(b, p_, tp_, pp_);
    }

private:
    CostParams p_;
    int tp_, pp_;
};

enum class Ev { Arrival, BatchStart, StageStart, StageEnd, TokenEmit, RequestFinish, Bubble };
enum class Bubble { PB1, PB2, PB3 };

struct Event {
    TimeUs t = 0;
    std::int64_t seq = 0;
    Ev kind = Ev::Arrival;
    int rid = -1, mb = -1, stage = -1, token = -1;
    TimeUs b_start = 0, b_end = 0;
    Bubble cls = Bubble::PB1;
};

struct MbSummary {  // engine.hpp:41-46
    std::int64_t prefill_tokens = 0;
    std::int64_t decode_kv = 0;
    bool decode_only() const { return prefill_tokens == 0; }
};

struct BubbleRec {
    int stage = 0;
    TimeUs start = 0, end = 0;
    Bubble cls = Bubble::PB1;
};

Bubble classify(const MbSummary& prev, const MbSummary& next);  // engine.cpp:32-40

// In-order pipeline occupancy (engine.cpp:42-81).
class Pipeline {
public:
    Pipeline(int stages, TimeUs send_us);
    struct Issue {
        std::vector<TimeUs> start, end;
        std::vector<BubbleRec> bubbles;
    };
    Issue advance(TimeUs issue, TimeUs stage_us, const MbSummary& s);
    TimeUs first_free() const { return busy_until_[0]; }
    const std::vector<TimeUs>& busy() const { return busy_; }

private:
    struct Last {
        bool exists = false;
        TimeUs end = 0;
        MbSummary s;
    };
    TimeUs send_us_;
    std::vector<TimeUs> busy_until_, busy_;
    std::vector<Last> last_;
};

struct MbRecord {
    int id = -1;
    TimeUs issue = 0, stage_us = 0, exit = 0;
    double iteration_ms = 0.0;
    std::vector<Entry> entries;
    MbSummary summary;
    std::int64_t total_tokens = 0;
};

struct SimOptions {
    bool keep_events = true;
    std::int64_t max_events = 50'000'000;
    bool check_block_tables = false;
};

struct Report {
    std::vector<Request> requests;
    std::vector<TimeUs> first_sched;
    std::vector<Event> events;
    std::vector<MbRecord> mbs;
    std::vector<BubbleRec> bubbles;
    std::vector<TimeUs> stage_busy;
    TimeUs makespan = 0;
    std::int64_t output_tokens = 0;
    std::int64_t peak_blocks = 0;

    std::string event_log_jsonl() const;  // byte-identical to engine.cpp:332-371
};

Report simulate(const ReplicaConfig& cfg, const CostParams& params, const std::vector<Request>& trace,
                StepExecutor& exec, const SimOptions& opts = {});

}  // namespace ss
