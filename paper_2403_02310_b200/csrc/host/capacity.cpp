#include "capacity.hpp"

#include <algorithm>
#include <thread>

namespace ss {

bool meets_slo(const Latency& r, double slo_ms, double max_sched_delay_ms) {
    return r.tbt_p99_ms <= slo_ms && r.sched_delay_median_ms <= max_sched_delay_ms;
}

CapacityResult capacity_search(const Probe& probe, double slo_ms, const CapacityOptions& o) {
    auto measure = [&](double qps) {
        CapacityProbe p;
        p.qps = qps;
        p.report = probe(qps);
        p.pass = meets_slo(p.report, slo_ms);
        return p;
    };
    // Rungs qps_low * 2^k <= max_qps: a fixed grid, so the answer does not
    // depend on how many rungs run at once.
    std::vector<double> rungs{o.qps_low};
    while (rungs.back() * 2.0 <= o.max_qps) rungs.push_back(rungs.back() * 2.0);

    std::vector<CapacityProbe> got(rungs.size());
    std::size_t probed = 0;
    int fail_at = -1;
    const std::size_t width = std::size_t(std::max(1, o.parallel));
    while (probed < rungs.size() && fail_at < 0) {
        const std::size_t n = std::min(width, rungs.size() - probed);
        if (n == 1) {
            got[probed] = measure(rungs[probed]);
        } else {
            std::vector<std::thread> pool;
            for (std::size_t i = 0; i < n; ++i)
                pool.emplace_back([&, i] { got[probed + i] = measure(rungs[probed + i]); });
            for (std::thread& t : pool) t.join();
        }
        for (std::size_t i = probed; i < probed + n; ++i)
            if (!got[i].pass) {
                fail_at = int(i);
                break;
            }
        probed += n;
    }
    CapacityResult res;
    res.probes.assign(got.begin(), got.begin() + std::ptrdiff_t(probed));
    if (fail_at == 0) throw InfeasibleSlo("qps_low fails the SLO");

    double lo = rungs.back(), hi = rungs.back();  // never failed: report the cap
    if (fail_at > 0) {
        lo = rungs[std::size_t(fail_at) - 1];
        hi = rungs[std::size_t(fail_at)];
    }
    while (hi - lo > o.rel_width * hi) {
        const double mid = 0.5 * (lo + hi);
        res.probes.push_back(measure(mid));
        (res.probes.back().pass ? lo : hi) = mid;
    }
    double best = 0;
    for (const CapacityProbe& p : res.probes)
        if (p.pass) best = std::max(best, p.qps);
    for (const CapacityProbe& p : res.probes)
        if (!p.pass && p.qps < best) res.monotone_warning = true;
    res.qps = best;
    return res;
}

}  // namespace ss
