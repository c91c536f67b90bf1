// Latency summary of a run: nearest-rank percentiles, TTFT/TBT/scheduling
// delay with a warm-up exclusion, throughput and bubble fraction. Restates
// reference proj/src/metrics.cpp:13-68.
#pragma once

#include <vector>

#include "engine.hpp"

namespace ss {

struct Latency {
    double ttft_median_ms = 0, tbt_p99_ms = 0, tbt_median_ms = 0, sched_delay_median_ms = 0;
    double throughput_tps = 0, bubble_fraction = 0, makespan_ms = 0;
    std::int64_t tbt_samples = 0;
    int n_requests = 0;
};

double percentile(std::vector<double> v, double p);  // index ceil(p/100*n)-1 of the sorted series
Latency summarize(const Report& rep, double warmup_frac = 0.05);

struct Slo {
    double strict_ms = 0, relaxed_ms = 0;  // 5x / 25x the 32x4k decode iteration
};
Slo slo_for(const CostParams& p);

}  // namespace ss
