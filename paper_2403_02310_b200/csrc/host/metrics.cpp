#include "metrics.hpp"

#include <algorithm>
#include <cmath>

namespace ss {

double percentile(std::vector<double> v, double p) {
    if (v.empty()) throw ContractViolation("percentile of empty series");
    if (p < 0.0 || p > 100.0) throw ContractViolation("percentile rank out of range");
    std::sort(v.begin(), v.end());
    const auto n = std::int64_t(v.size());
    const std::int64_t rank = std::int64_t(std::ceil(p / 100.0 * double(n))) - 1;
    return v[std::size_t(std::clamp<std::int64_t>(rank, 0, n - 1))];
}

Latency summarize(const Report& rep, double warmup_frac) {
    Latency L;
    const int n = int(rep.requests.size());
    L.n_requests = n;
    L.makespan_ms = us_to_ms(rep.makespan);
    // The first warmup_frac of requests (by arrival index) carry cold-start
    // bias and are excluded from the latency series.
    const int skip = int(std::floor(warmup_frac * n));
    std::vector<double> ttft, tbt, delay;
    for (int i = skip; i < n; ++i) {
        const Request& r = rep.requests[std::size_t(i)];
        if (r.first_token) ttft.push_back(us_to_ms(*r.first_token - r.arrival));
        if (rep.first_sched[std::size_t(i)] >= 0) delay.push_back(us_to_ms(rep.first_sched[std::size_t(i)] - r.arrival));
        for (std::size_t k = 1; k < r.emits.size(); ++k) tbt.push_back(us_to_ms(r.emits[k] - r.emits[k - 1]));
    }
    if (!ttft.empty()) L.ttft_median_ms = percentile(ttft, 50);
    if (!delay.empty()) L.sched_delay_median_ms = percentile(delay, 50);
    L.tbt_samples = std::int64_t(tbt.size());
    if (!tbt.empty()) {
        L.tbt_p99_ms = percentile(tbt, 99);
        L.tbt_median_ms = percentile(tbt, 50);
    }
    if (rep.makespan > 0) L.throughput_tps = double(rep.output_tokens) / (us_to_ms(rep.makespan) / 1000.0);
    std::int64_t bubble_us = 0;
    for (const BubbleRec& b : rep.bubbles) bubble_us += b.end - b.start;
    const auto stages = std::int64_t(rep.stage_busy.size());
    if (rep.makespan > 0 && stages > 0)
        L.bubble_fraction = double(bubble_us) / (double(rep.makespan) * double(stages));
    return L;
}

Slo slo_for(const CostParams& p) {
    const double ref = decode_reference_time(p);
    return Slo{5.0 * ref, 25.0 * ref};
}

}  // namespace ss
