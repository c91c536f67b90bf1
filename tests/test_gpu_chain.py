"""The fused projection chain (SS_CHAIN=1: layer l's O -> gate/up -> down and layer l + 1's
QKV in one persistent launch with per-tile ready flags; gemm.cu gemm_chain_kernel).

Opt-in (measured slower than the separate launches on the canonical batch),
so these tests keep it correct: with whole tiles (no K splits) every output tile is the same
sequence of MMAs as the separate kernels' whole-tile schedule, so the logits must be
bitwise equal; with K splits (fixed-order fp32 reduction of the split partials) the forward
must meet the oracle tolerance and be bitwise repeatable.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2403_02310_b200 import gpu, host  # noqa: E402

from test_gpu_forward import compare, orc_mod  # noqa: E402

pytestmark = pytest.mark.gpu


def forward(shape, d, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:  # the tuning is read once at ss_create
        f = gpu.HybridForward(shape, weight_seed=1234)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    f.kv_alloc(d.pool_blocks)
    f.fill_descriptor_prefixes(d, seed=5)
    a, _, _ = f.forward(d)
    b, _, _ = f.forward(d)
    f.set_profiling(True)
    f.kernel_times(reset=True)
    f.forward(d)
    kt = f.kernel_times(reset=True)
    f.close()
    return a, b, kt


def test_chain_whole_tiles_bitwise_equal_to_separate_launches():
    s = gpu.MODELS["mistral7b"].with_layers(2)
    # M = 2048: every phase has >= 74 tiles; SS_GEMM_SK=0 forces the separate kernels'
    # whole-tile schedule too, so both paths run the same MMA sequence per tile
    d = host.Descriptor.canonical(2048, 32, 4096, 0, vocab=s.vocab, token_seed=3)
    ref, _, kt0 = forward(s, d, {"SS_CHAIN": "0", "SS_GEMM_QKV": "0,256", "SS_GEMM_O": "0,256",
                                 "SS_GEMM_GATEUP": "0,256", "SS_GEMM_DOWN": "0,256"})
    out, out2, kt = forward(s, d, {"SS_CHAIN": "1", "SS_CHAIN_S": "1,1,1,1"})
    assert kt["gemm_chain"][1] == 2 and kt["gemm_gate_up"][1] == 0, kt
    assert kt0["gemm_chain"][1] == 0
    assert np.array_equal(out, out2)
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("tau,splits", [(512, "0,0,0,0"), (512, "2,1,4,2"), (300, "1,1,3,1")])
def test_chain_split_k_matches_oracle(tau, splits):
    s = gpu.MODELS["mistral7b"].with_layers(2)
    d = host.Descriptor.canonical(tau, 32, 4096, 0, vocab=s.vocab, token_seed=3)
    out, out2, kt = forward(s, d, {"SS_CHAIN": "1", "SS_CHAIN_S": splits})
    assert kt["gemm_chain"][1] == 2, kt
    assert np.array_equal(out, out2)  # fixed split order: deterministic
    o = orc_mod.Oracle(s, weight_seed=1234, num_blocks=d.pool_blocks)
    o.fill_descriptor_prefixes(d, seed=5)
    ref = o.forward(d)
    o.close()
    compare(out, ref, f"chain tau={tau} splits={splits}", "full_width_2l")
