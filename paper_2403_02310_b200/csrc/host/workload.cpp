#include "workload.hpp"

#include <algorithm>
#include <cmath>

namespace ss {

namespace {
constexpr double kZ90 = 1.2816;  // standard-normal 90th percentile
constexpr double kTwoPi = 2.0 * 3.14159265358979323846;
}  // namespace

double Rng::uniform() {
    const std::uint64_t mant = gen_() >> 11;  // 53 random bits
    return (double(mant) + 0.5) * (1.0 / 9007199254740992.0);
}

double Rng::normal() {
    if (spare_ok_) {
        spare_ok_ = false;
        return spare_;
    }
    const double u1 = uniform();
    const double u2 = uniform();
    const double radius = std::sqrt(-2.0 * std::log(u1));
    const double angle = kTwoPi * u2;
    spare_ = radius * std::sin(angle);
    spare_ok_ = true;
    return radius * std::cos(angle);
}

double Rng::exponential(double mean) { return -mean * std::log(uniform()); }

int LogNormalLen::draw(Rng& rng) const {
    if (p90 < median) throw ContractViolation("p90 must be >= median");
    const double mu = std::log(median);
    const double sigma = (std::log(p90) - std::log(median)) / kZ90;
    const double v = std::exp(mu + sigma * rng.normal());
    return std::max(1, int(std::llround(v)));
}

std::optional<WorkloadSpec> workload_preset(const std::string& name) {
    if (name == "openchat") return WorkloadSpec{"openchat", {1730, 5696}, {415, 834}, 8192};
    if (name == "arxiv") return WorkloadSpec{"arxiv", {7059, 12985}, {208, 371}, 16384};
    return std::nullopt;
}

std::vector<Request> make_trace(const WorkloadSpec& spec, double qps, int n, std::uint64_t seed) {
    if (qps <= 0) throw ContractViolation("qps must be positive");
    Rng lengths(seed);
    Rng arrivals(seed ^ 0x9e3779b97f4a7c15ull);
    const double mean_gap_us = 1e6 / qps;
    std::vector<TimeUs> at(std::size_t(std::max(n, 0)));
    TimeUs t = 0;
    for (int i = 0; i < n; ++i) {
        t += std::max<TimeUs>(1, TimeUs(std::llround(arrivals.exponential(mean_gap_us))));
        at[std::size_t(i)] = t;
    }
    std::vector<Request> trace;
    trace.reserve(at.size());
    for (int i = 0; i < n; ++i) {
        int p = 0, o = 0;
        do {  // redraw the pair while it exceeds the total-length cap
            p = spec.prompt.draw(lengths);
            o = spec.output.draw(lengths);
        } while (std::int64_t(p) + o > spec.max_total);
        trace.emplace_back(i, at[std::size_t(i)], p, o);
    }
    return trace;
}

}  // namespace ss
