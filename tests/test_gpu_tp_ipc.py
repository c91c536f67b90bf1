"""Tensor-parallel forward over the CUDA-IPC transport, one process per rank.

Two processes (the round's boxes expose one B200, so both ranks share cuda:0; CUDA IPC
and the peer-memory kernels are the same across devices) create their rank contexts
without an NCCL id, exchange their exchange-region handles over a gloo process group
(ss_ipc_export / ss_ipc_open) and run the sharded forward: the O / down partials are
summed over peer memory by the fused all-reduce + residual-add kernel and the vocab
shards gathered by the logits kernel. Parity is against the fp32 oracle at TP1 with
test_gpu_forward's tolerance; repeated forwards (eager, graph capture, graph replays) must
agree bitwise (the fixed rank-order sum).
"""
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

pytest.importorskip("torch")

from paper_2403_02310_b200 import gpu, host  # noqa: E402

orc_mod = pytest.importorskip("oracle.forward")
from test_gpu_forward import compare  # noqa: E402

pytestmark = pytest.mark.gpu

TINY_TP = gpu.ModelShape("tiny_tp", 2, 256, 8, 4, 64, 1024, 512)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, q, tau, prefix, algo="auto"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        f = gpu.HybridForward(TINY_TP, tp_rank=rank, tp_size=world, nccl_id=None, weight_seed=1234, device=0)

        def allgather(b):
            out = [None] * world
            dist.all_gather_object(out, b)
            return out

        f.ipc_connect(allgather, max_tokens=4096)
        f.set_tp_allreduce(algo)
        d = host.Descriptor.canonical(tau, 32, 4096, prefix, vocab=TINY_TP.vocab, token_seed=7)
        f.kv_alloc(d.pool_blocks)
        f.fill_descriptor_prefixes(d, seed=5)
        lg, nt, _ = f.forward(d)
        # forward 2 captures the CUDA graph, 3 and 4 replay it (fresh collective epochs)
        for _ in range(3):
            lg2, nt2, _ = f.forward(d)
            assert np.array_equal(lg, lg2) and np.array_equal(nt, nt2), "IPC TP forward is not deterministic"
        assert f.graph_stats() == (1, 2), f.graph_stats()
        dist.barrier()  # every rank done reading peer memory before any unmaps
        f.close()
        q.put((rank, lg, nt, lg2, nt2, None))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, None, None, None, None, repr(e)))
    finally:
        dist.destroy_process_group()


def _run(world, tau, prefix, algo):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, q, tau, prefix, algo)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, lg, nt, lg2, nt2, err = q.get(timeout=600)
        res[r] = (lg, nt, lg2, nt2, err)
    for p in procs:
        p.join(timeout=120)
    for r in range(world):
        assert res[r][4] is None, f"rank {r}: {res[r][4]}"
    lg, nt, lg2, nt2, _ = res[0]
    assert np.array_equal(lg, lg2) and np.array_equal(nt, nt2), "IPC TP forward is not deterministic"
    for r in range(1, world):
        assert np.array_equal(lg, res[r][0]), f"ranks 0 and {r} disagree on the gathered logits"
    assert (nt == lg.argmax(1)).all()
    d = host.Descriptor.canonical(tau, 32, 4096, prefix, vocab=TINY_TP.vocab, token_seed=7)
    o = orc_mod.Oracle(TINY_TP, weight_seed=1234, num_blocks=d.pool_blocks)
    o.fill_descriptor_prefixes(d, seed=5)
    compare(lg, o.forward(d), f"tiny tp{world} ipc {algo} tau={tau} prefix={prefix}")
    return lg


@pytest.mark.parametrize("tau,prefix", [(512, 0), (512, 2048)])
def test_tiny_tp2_ipc_vs_oracle(tau, prefix):
    _run(2, tau, prefix, "auto")


@pytest.mark.parametrize("world", [2, 4])
def test_tp_ipc_two_shot(world):
    """Reduce-scatter + all-gather over peer memory (the 8-GPU algorithm): parity with the
    oracle, identical logits on every rank, deterministic; tp=4 four processes."""
    two = _run(world, 512, 0, "twoshot")
    one = _run(world, 512, 0, "oneshot")
    # same sums up to the bf16 rounding of each rank's reduced share
    assert np.abs(two - one).max() <= 2e-2 * np.abs(one).max()


@pytest.mark.parametrize("world,tau", [(2, 512), (4, 512), (4, 40)])
def test_tp_ipc_push_equals_two_shot(world, tau):
    """Reduce-scatter fused into the O / down GEMM epilogue (every unit stored into its owner
    rank's landing zone, the reduction reading local memory): bitwise the two-shot result,
    since both sum the same bf16 partials in rank order; and the auto pick at tp=4."""
    push = _run(world, tau, 0, "push")
    two = _run(world, tau, 0, "twoshot")
    assert np.array_equal(push, two), f"push vs two-shot: max diff {np.abs(push - two).max()}"
    if world == 4 and tau == 512:  # 512 x 256 x 2 B < 1 MB: auto stays one-shot on the tiny shape
        assert np.array_equal(_run(world, 512, 0, "auto"), _run(world, 512, 0, "oneshot"))
