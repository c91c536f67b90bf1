// Capacity under an SLO — the paper's headline metric and
// SURVEY §8f-2. Restates servesim::capacity_search and meets_slo (reference
// proj/src/metrics.cpp:65-138, metrics.hpp:41-70): a doubling ladder of qps
// from qps_low (probed `parallel` at a time, the reference's OpenMP chunking)
// up to the first failing rung, then sequential bisection to rel_width. A
// probe passes when P99 TBT <= slo and the median scheduling delay <= 2 s.
//
// The probe is any deterministic function of qps: the reference clock
// (CostModelExecutor), a calibrated B200 clock, or real B200 forwards
// (GpuExecutor, then parallel must be 1).
#pragma once

#include <functional>
#include <vector>

#include "metrics.hpp"

namespace ss {

bool meets_slo(const Latency& r, double slo_ms, double max_sched_delay_ms = 2000.0);

struct CapacityOptions {  // metrics.hpp:45-49
    double qps_low = 0.01;
    double max_qps = 1024.0;
    double rel_width = 0.05;
    int parallel = 1;  // ladder rungs probed concurrently (reference: omp_get_max_threads())
};

struct CapacityProbe {
    double qps = 0;
    bool pass = false;
    Latency report;
};

struct CapacityResult {
    double qps = 0;                 // highest passing probe
    bool monotone_warning = false;  // a failing probe below a passing one
    std::vector<CapacityProbe> probes;
};

using Probe = std::function<Latency(double qps)>;

// Throws InfeasibleSlo when qps_low fails.
CapacityResult capacity_search(const Probe& probe, double slo_ms, const CapacityOptions& opts = {});

}  // namespace ss
