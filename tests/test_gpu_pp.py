"""Pipeline parallelism on the GPU path (reference engine.cpp:42-81 and the
stage model behind iteration_time(..., pp), costmodel.cpp:55).

Stage s of pp holds layers [s*L/pp, (s+1)*L/pp) with their global synthetic weights and
caches; the residual stream is handed from stage to stage. Every stage runs the same kernels
on the same data as the unpipelined forward, so the logits must be bitwise equal to PP = 1.
The restated engine then runs the stall-free schedule with the pipeline as its model step.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2403_02310_b200 import _lib, gpu, host  # noqa: E402

pytestmark = pytest.mark.gpu


def pp1(shape, d):
    f = gpu.HybridForward(shape, weight_seed=1234)
    f.kv_alloc(d.pool_blocks)
    f.fill_descriptor_prefixes(d, seed=5)
    lg, nt, _ = f.forward(d)
    f.close()
    return lg, nt


@pytest.mark.parametrize("model,layers,pp", [("tiny", 2, 2), ("mistral7b", 4, 2), ("mistral7b", 4, 4),
                                             ("mistral7b", 5, 2)])
@pytest.mark.parametrize("batch", ["canonical", "prefix2048", "decode"])
def test_pipeline_bitwise_equal_to_unpipelined(model, layers, pp, batch):
    s = gpu.MODELS[model].with_layers(layers)
    if batch == "decode":
        d = host.Descriptor.build([host.BatchEntry(i, "decode", 1, 3000 + 64 * i) for i in range(12)], vocab=s.vocab,
                                  token_seed=3)
    else:
        d = host.Descriptor.canonical(512, 32, 4096, 2048 if batch == "prefix2048" else 0, vocab=s.vocab, token_seed=3)
    ref, ref_nt = pp1(s, d)
    g = gpu.PipelineGroup(s, pp, weight_seed=1234)
    g.kv_alloc(d.pool_blocks)
    g.fill_descriptor_prefixes(d, seed=5)
    lg, nt, _ = g.forward(d)
    lg2, _, ms = g.forward(d)
    assert len(g.stage_ms) == pp and all(t > 0 for t in g.stage_ms) and ms == max(g.stage_ms)
    g.close()
    assert np.array_equal(lg, ref), float(np.abs(lg - ref).max())
    assert np.array_equal(nt, ref_nt)
    assert np.array_equal(lg2, ref)  # the hand-off buffers are reused safely across forwards


def test_stage_contexts_hold_their_layers_only():
    s = gpu.MODELS["tiny"].with_layers(4)
    g = gpu.PipelineGroup(s, 2)
    g.stages[0].weight("embed")
    with pytest.raises(_lib.SSError):
        g.stages[1].weight("embed")
    with pytest.raises(_lib.SSError):
        g.stages[0].weight("lm_head")
    g.stages[1].weight("lm_head")
    g.close()
    with pytest.raises(_lib.SSError):
        gpu.PipelineGroup(s, 5)  # more stages than layers


def test_engine_closed_loop_on_pipeline_stages():
    s = gpu.MODELS["tiny"].with_layers(4)
    g = gpu.PipelineGroup(s, 2)
    g.kv_alloc(4096)
    trace = host.make_trace("openchat", 4.0, 8, 42)
    params = host.model_preset("tiny")
    cfg = host.ReplicaConfig(token_budget=512, kv_blocks=4096, pp_degree=2)
    rep = host.simulate(cfg, params, trace, gpu=g, token_seed=1, keep_events=False)
    mbs = list(rep.microbatches())
    assert len(mbs) > 0 and all(mb.iteration_ms > 0 for mb in mbs)
    # the engine's pipeline model: iteration = stages x the per-stage (slowest stage) time
    last = mbs[-1]
    g.forward(host.Descriptor.build(last.entries, vocab=s.vocab, token_seed=1), logits=False)
    assert last.iteration_ms == pytest.approx(2 * max(g.stage_ms), rel=0.5)
    summ = rep.summarize()
    assert summ["n_requests"] == 8 and summ["tbt_p99_ms"] > 0
    # a pipeline model step needs pp_degree == stages
    with pytest.raises(_lib.ContractViolation):
        host.simulate(host.ReplicaConfig(token_budget=512, kv_blocks=4096, pp_degree=1), params, trace, gpu=g)
    g.close()
