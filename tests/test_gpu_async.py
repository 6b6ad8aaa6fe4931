"""The barrier-free traversal (DFGTB_TRAV_ASYNC=1) against the level-synchronous one
(default): every entry's arithmetic and every item's (key, rank) are the same, so the
sums, statistics and CV scores must be bit-identical."""
import os

import numpy as np
import pytest

from paper_1102_2878_b200 import datagen

pytestmark = pytest.mark.gpu


def _engine(dfgtb, x, levels, **kw):
    if not levels:
        os.environ["DFGTB_TRAV_ASYNC"] = "1"
    try:
        return dfgtb.DualTreeEngine(x, config=dfgtb.EngineConfig(leaf_threshold=32, **kw))
    finally:
        os.environ.pop("DFGTB_TRAV_ASYNC", None)


@pytest.mark.parametrize("k,scale", [(1, 1.0), (2, 0.2), (3, 0.05), (4, 0.05)])
def test_async_equals_levels(dfgtb, k, scale):
    w = datagen.config(k, scale)
    hs = [s * w.h_s for s in w.scales] + [2 * s * w.h_s for s in w.scales]
    ea, el = _engine(dfgtb, w.refs, False), _engine(dfgtb, w.refs, True)
    ga, gl = ea.compute_batch(None, hs), el.compute_batch(None, hs)
    assert np.array_equal(ga, gl)
    for sa, sl in zip(ea.batch_stats(), el.batch_stats()):
        for f in ("kernel_evaluations", "pairs_visited", "base_cases", "prunes_finite_diff",
                  "prunes_farfield", "prunes_direct_local", "prunes_far_to_local", "levels",
                  "pairs_covered"):
            assert getattr(sa, f) == getattr(sl, f), f
    ra, rl = ea.sweep(w.scales, w.h_s), el.sweep(w.scales, w.h_s)
    for a, b in zip(ra, rl):
        assert (a.lk_score, a.lk_clamped, a.ls_score) == (b.lk_score, b.lk_clamped, b.ls_score)


def test_async_queries_and_overflow_regrowth(dfgtb):
    # Q != R, and a first batch whose buffers must grow (big bandwidth batch)
    r = datagen.clustered_3d(20000, 77)
    q = np.random.default_rng(3).random((15000, 3))
    hs = datagen.silverman_h(r) * np.geomspace(0.05, 20, 40)
    ea, el = _engine(dfgtb, r, False), _engine(dfgtb, r, True)
    assert np.array_equal(ea.compute_batch(q, hs), el.compute_batch(q, hs))
