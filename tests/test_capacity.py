"""Capacity under an SLO: capacity_search restated in libss_host.so,
checked live against the compiled reference (servesim::capacity_search with the
CLI probe, metrics.cpp:70-138, cli.cpp:434-439): identical capacity, identical
probe sequence (qps, pass) and identical per-probe latency summaries. (The
reference is built here without OpenMP, i.e. one ladder rung at a time; with
concurrent rungs our probe list is a superset, as the reference's own comment
at metrics.cpp:80 allows.)"""
import pytest

from paper_2403_02310_b200 import _lib, host

ref = pytest.importorskip("oracle.ref")
needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built (reference tree absent)")


def _cfg(policy, tau=512):
    c = host.ReplicaConfig()
    c.scheduler = policy
    c.token_budget = tau
    return c


@needs_ref
@pytest.mark.parametrize("policy,model,workload,slo", [
    ("stall_free", "yi34b", "openchat", "strict"), ("vllm", "yi34b", "openchat", "relaxed"),
    ("stall_free", "mistral7b", "arxiv", "relaxed"), ("orca", "mistral7b", "openchat", "strict"),
])
@pytest.mark.parametrize("parallel", [1, 3])
def test_capacity_matches_reference(policy, model, workload, slo, parallel):
    p = host.model_preset(model)
    strict, relaxed = host.slo_thresholds(p)
    slo_ms = strict if slo == "strict" else relaxed
    cfg = _cfg(policy)
    kw = dict(qps_low=0.05, max_qps=32.0, rel_width=0.1, parallel=parallel)
    try:
        ours = host.capacity_search(cfg, p, workload, 96, 17, slo_ms, **kw)
        ours_err = None
    except _lib.InfeasibleSlo as e:
        ours, ours_err = None, e
    st, qps, mono, probes = ref.capacity(cfg._c(), p._c(), workload, 96, 17, slo_ms,
                                         _lib.CapacityOpts(kw["qps_low"], kw["max_qps"], kw["rel_width"], parallel))
    if ours_err is not None:
        assert st == _lib.SS_INFEASIBLE
        return
    assert st == 0
    assert ours.qps == qps and ours.monotone_warning == mono
    mine = [(q.qps, q.passed, q.report) for q in ours.probes]
    if parallel == 1:
        assert mine == probes
    else:  # concurrent rungs may probe past the first failure; the answer is grid-fixed
        assert all(p in mine for p in probes)


def test_capacity_infeasible_and_cap():
    p = host.model_preset("mistral7b")
    cfg = _cfg("stall_free")
    with pytest.raises(_lib.InfeasibleSlo):
        host.capacity_search(cfg, p, "openchat", 32, 1, 1e-3, qps_low=0.5, max_qps=4.0)
    r = host.capacity_search(cfg, p, "openchat", 32, 1, 1e9, qps_low=0.5, max_qps=4.0)
    assert r.qps == 4.0 and all(q.passed for q in r.probes) and [q.qps for q in r.probes] == [0.5, 1.0, 2.0, 4.0]
