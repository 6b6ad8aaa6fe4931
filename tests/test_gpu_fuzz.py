"""Seeded random sweep over the engine's input space (sizes, dimensions, leaf sizes,
bandwidths, epsilons, Q != R, batch sizes, duplicates): every query within eps of the
oracle's exact sum.  Exercises the sync-free batch (first batches overflow and rerun),
the two-stream execution, the MUFU / FP64 exp switch and the generic D > 5 path."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _case(seed):
    g = np.random.default_rng(seed)
    d = int(g.choice([1, 2, 2, 3, 3, 4, 5, 6]))
    n = int(g.integers(1, 3000))
    kind = g.integers(0, 3)
    if kind == 0:
        x = g.random((n, d))
    elif kind == 1:  # clusters + exact duplicates
        c = g.random((max(1, n // 50), d))
        x = c[g.integers(0, len(c), n)] + 0.01 * g.standard_normal((n, d))
        x[: n // 10] = x[0]
    else:  # anisotropic
        x = g.random((n, d)) * (10.0 ** g.uniform(-3, 1, size=d))
    q = None if g.random() < 0.5 else g.random((int(g.integers(1, 800)), d)) * x.max(axis=0)
    eps = float(g.choice([0.0, 1e-3, 1e-2, 0.1, 0.5]))
    leaf = int(g.choice([1, 4, 16, 32, 64]))
    span = float(np.max(x.max(axis=0) - x.min(axis=0))) or 1.0
    hs = list(span * 10.0 ** g.uniform(-4, 1, size=int(g.integers(1, 6))))
    return x, q, eps, leaf, hs


@pytest.mark.parametrize("seed", range(200))
def test_random_inputs_meet_eps(dfgtb, orc, seed):
    x, q, eps, leaf, hs = _case(seed)
    cfg = dfgtb.EngineConfig(epsilon=eps, leaf_threshold=leaf)
    with dfgtb.DualTreeEngine(x, dfgtb.Mode.series, cfg) as e:
        got = e.compute_batch(q, hs)
        again = e.compute_batch(q, hs)
    assert np.array_equal(got, again)  # deterministic, overflow reruns included
    qq = x if q is None else q
    for b, h in enumerate(hs):
        ex = orc.naive_kde(qq, x, h)
        ok = ex > 0
        # eps = 0: exact up to rounding; terms exp(-y) with y up to ~745 carry relative
        # error ~y * 1e-15 from the rounding of y itself (both here and in the oracle)
        tol = max(eps, 1e-10)
        err = np.abs(got[b][ok] - ex[ok]) - tol * ex[ok] * (1 + 1e-12) - 1e-300
        if np.any(err > 0):
            i = int(np.argmax(err))
            raise AssertionError(f"seed {seed} h {h} eps {eps} leaf {leaf} n {x.shape} q {None if q is None else q.shape}: "
                                 f"got {got[b][ok][i]!r} exact {ex[ok][i]!r}")
        assert np.all(got[b][~ok] <= 1e-300)
