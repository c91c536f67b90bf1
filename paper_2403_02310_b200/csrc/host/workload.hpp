// Synthetic request traces, bit-identical to the reference's make_trace
// (reference proj/src/workload.cpp:16-84): mt19937_64 with explicit uniform,
// Box-Muller normal and exponential transforms, log-normal lengths from a
// (median, P90) pair with a rejection cap on prompt + output, Poisson arrivals
// from an independently seeded stream. Relies on the platform libm for
// log/exp/sin/cos exactly as the reference does.
#pragma once

#include <cstdint>
#include <random>
#include <string>
#include <optional>
#include <vector>

#include "types.hpp"

namespace ss {

class Rng {
public:
    explicit Rng(std::uint64_t seed) : gen_(seed) {}
    double uniform();  // (0, 1), 53 bits
    double normal();   // Box-Muller with a cached spare
    double exponential(double mean);

private:
    std::mt19937_64 gen_;
    bool spare_ok_ = false;
    double spare_ = 0.0;
};

struct LogNormalLen {  // workload.hpp:31-39
    double median = 1;
    double p90 = 1;
    int draw(Rng& rng) const;
};

struct WorkloadSpec {
    std::string name;
    LogNormalLen prompt, output;
    std::int64_t max_total = 8192;
};

std::optional<WorkloadSpec> workload_preset(const std::string& name);  // presets.cpp:82-100
std::vector<Request> make_trace(const WorkloadSpec& spec, double qps, int n, std::uint64_t seed);

}  // namespace ss
