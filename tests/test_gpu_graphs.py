"""CUDA graphs of the forward (ss_set_graphs): a captured-and-replayed forward is bitwise
identical to eager launches, across repeated shapes (replays), alternating shapes (one
graph each), workspace growth (graphs invalidated and re-captured) and the stream-K GEMM
schedules whose ready flags carry per-forward epochs (EpiArgs::epoch_base).

The graph is the engine.cpp:227 model step made one launch: the closed-loop engine calls
the forward once per iteration with a new descriptor of a recurring shape.
"""
import numpy as np
import pytest

pytest.importorskip("torch")

from paper_2403_02310_b200 import gpu, host  # noqa: E402

pytestmark = pytest.mark.gpu


def _pair(shape, pool):
    """Two contexts with identical weights and caches: eager and graph-replayed."""
    ctxs = []
    for graphs in (False, True):
        f = gpu.HybridForward(shape, weight_seed=1234)
        f.set_graphs(graphs)
        f.kv_alloc(pool)
        ctxs.append(f)
    return ctxs


def _fill(ctxs, d):
    for f in ctxs:
        f.fill_descriptor_prefixes(d, seed=5)


@pytest.mark.parametrize("model", ["tiny", "mistral7b"])
def test_graph_replay_bitwise(model):
    """Repeated canonical batches (Mistral at 2 layers: M=512 stream-K gate/up and down,
    whose cross-CTA flags need fresh epochs on every replay)."""
    s = gpu.MODELS[model] if model == "tiny" else gpu.MODELS[model].with_layers(2)
    d = host.Descriptor.canonical(512, 32, 4096, 0, vocab=s.vocab, token_seed=7)
    eager, graphed = _pair(s, d.pool_blocks)
    _fill([eager, graphed], d)
    for _ in range(5):
        le, ne, _ = eager.forward(d)
        lg, ng, _ = graphed.forward(d)
        assert np.array_equal(le, lg) and np.array_equal(ne, ng)
    cap, rep = graphed.graph_stats()
    assert cap == 1 and rep == 3, (cap, rep)  # eager, capture (+launch), 3 replays
    assert eager.graph_stats() == (0, 0)
    # launch accounting covers replayed kernels
    assert graphed.launch_count == eager.launch_count
    eager.close()
    graphed.close()


def test_graph_alternating_shapes_and_growth():
    """Decode-only, hybrid and prefix-2048 batches interleaved (one graph per shape), then a
    larger batch that reallocates the workspaces (every graph dropped and re-captured)."""
    s = gpu.MODELS["tiny"]
    ds = [
        host.Descriptor.build([host.BatchEntry(i, "decode", 1, 4095 + 17 * i) for i in range(32)],
                              vocab=s.vocab, token_seed=3),
        host.Descriptor.canonical(512, 32, 4096, 0, vocab=s.vocab, token_seed=7),
        host.Descriptor.canonical(512, 32, 4096, 2048, vocab=s.vocab, token_seed=9),
    ]
    big = host.Descriptor.canonical(2048, 32, 4096, 0, vocab=s.vocab, token_seed=11)
    pool = max(x.pool_blocks for x in ds + [big])
    eager, graphed = _pair(s, pool)
    for seq in (ds * 3, [big, big, big] + ds * 2):
        for d in seq:
            _fill([eager, graphed], d)
            le, ne, _ = eager.forward(d)
            lg, ng, _ = graphed.forward(d)
            assert np.array_equal(le, lg) and np.array_equal(ne, ng)
    cap, rep = graphed.graph_stats()
    assert cap >= 4 and rep >= 5, (cap, rep)
    eager.close()
    graphed.close()


def test_graph_trace_steps_match_eager():
    """Closed-loop style: 300 consecutive micro-batches of a simulated stall-free stream
    through one session (KV appended every step, shapes recurring), eager vs graphs,
    bitwise."""
    s = gpu.MODELS["tiny"]
    trace = host.make_trace("openchat", 16, 24, 3)
    rep = host.simulate(host.ReplicaConfig(kv_blocks=20000), host.model_preset("tiny"), trace)
    sess = host.Session(20000, vocab=s.vocab, token_seed=42)
    eager, graphed = _pair(s, 20000)
    n = 0
    for mb, pl, done in host.replay_plan(rep, trace):
        d = sess.step(mb.entries, pl)
        le, _, _ = eager.forward(d)
        lg, _, _ = graphed.forward(d)
        assert np.array_equal(le, lg), f"step {n}"
        for r in done:
            sess.release(r)
        n += 1
        if n == 300:
            break
    assert n == 300
    assert graphed.graph_stats()[1] > 0
    eager.close()
    graphed.close()
