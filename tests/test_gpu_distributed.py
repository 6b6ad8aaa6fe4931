"""Query-sharded CV sweep with the GPU engine, ranks emulated in one
process on one GPU (the round's boxes have one GPU; no rank waits on another).

Each shard's sums come from DualTreeEngine(refs).compute_batch(shard_queries, hs)
(Q != R: a query tree per shard); the partial sums are added as the all_reduce
would.  Scores must agree with the single-engine sweep within the rigorous 2-eps
bound (both are eps-accurate per query, with different prune decisions).
"""
import numpy as np
import pytest

from paper_1102_2878_b200 import datagen
from paper_1102_2878_b200.distributed import sharded_sweep

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_sweep_matches_single_engine(dfgtb, orc, world):
    w = datagen.config(2, scale_n=0.04)
    refs, eps = w.refs, 0.01
    eng = dfgtb.DualTreeEngine(refs, config=dfgtb.EngineConfig(epsilon=eps, leaf_threshold=32))
    scales = w.scales[2:7]
    single = eng.sweep(scales, w.h_s)
    shards = []
    for rank in range(world):
        rows = sharded_sweep(refs, scales, w.h_s, lambda q, hs: eng.compute_batch(q, hs), rank, world,
                             lambda x: shards.append(x) or x)
    total = np.sum(shards, axis=0).reshape(len(scales), 3)
    n, d = refs.shape
    for k, (s, r1) in enumerate(zip(scales, single)):
        h = s * w.h_s
        lk, ls = total[k, 0] / n, total[k, 2] / n
        g1, g2 = orc.naive_kde(refs, refs, h), orc.naive_kde(refs, refs, 2 * h)
        nh = (n - 1) * (2 * np.pi * h * h) ** (d / 2)
        nc = (n - 1) * (2 * np.pi * 4 * h * h) ** (d / 2)
        bound = 2 * eps / n * np.sum(g2 / nc + 2 * g1 / nh) * (1 + 1e-9)
        assert abs(ls - r1.ls_score) <= bound
        kappa = np.max(2 * eps * g1 / np.maximum(g1 - 1.0, 1e-300))
        if kappa < 0.5:
            assert abs(lk - r1.lk_score) <= -np.mean(np.log1p(-2 * eps * g1 / (g1 - 1.0))) + 1e-15


def _gpu_worker(rank, world, port, out):
    """One rank of the bench's N > 1 path: the GPU engine's sums of this rank's tree-order
    query shard, CV partials all-reduced over gloo (NCCL on a multi-GPU node)."""
    import os

    import torch.distributed as dist

    import paper_1102_2878_b200 as dfgtb
    from paper_1102_2878_b200 import datagen
    from paper_1102_2878_b200.distributed import sharded_sweep, torch_allreduce
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = datagen.config(2, scale_n=0.1)
    eng = dfgtb.DualTreeEngine(w.refs, config=dfgtb.EngineConfig(epsilon=0.01, leaf_threshold=32))
    order = eng.reference_tree().perm
    rows = sharded_sweep(w.refs, w.scales, w.h_s, lambda q, hs: eng.compute_batch(q, hs), rank, world,
                         torch_allreduce(), order=order)
    out[rank] = [(r.h, r.lk_score, r.lk_clamped, r.ls_score) for r in rows]
    dist.barrier()
    dist.destroy_process_group()


def test_two_process_gloo_sweep_with_gpu_engines(dfgtb, orc):
    """Two processes (one GPU here; the kernels of the ranks never wait on each other), each
    sweeping its shard on the GPU, one gloo all_reduce of 3 partials per bandwidth: every
    rank gets the same rows, within the 2-eps bounds of the single-engine sweep."""
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    with mp.Manager() as man:
        out = man.dict()
        mp.spawn(_gpu_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    assert res[0] == res[1]
    w = datagen.config(2, scale_n=0.1)
    refs, eps = w.refs, 0.01
    n, d = refs.shape
    single = dfgtb.DualTreeEngine(refs, config=dfgtb.EngineConfig(epsilon=eps, leaf_threshold=32)).sweep(w.scales, w.h_s)
    for (h, lk, cl, ls), r1 in zip(res[0], single):
        assert abs(h - r1.h) <= 1e-15 * h
        g1, g2 = orc.naive_kde(refs, refs, h), orc.naive_kde(refs, refs, 2 * h)
        nh = (n - 1) * (2 * np.pi * h * h) ** (d / 2)
        nc = (n - 1) * (2 * np.pi * 4 * h * h) ** (d / 2)
        assert abs(ls - r1.ls_score) <= 2 * eps / n * np.sum(g2 / nc + 2 * g1 / nh) * (1 + 1e-9)
