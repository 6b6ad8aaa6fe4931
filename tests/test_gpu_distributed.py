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
