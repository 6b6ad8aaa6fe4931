"""CV scores on the device (K11) vs hand formulas and the reference.

Pins: test_cv.cpp:25-79 hand formulas incl. the golden -0.26698943846309625;
lkcv/lscv on identical sums match the oracle to 1e-12 relative (FP64 summation
order); DFGT-driven scores agree with the naive-driven ones within the
reference's own slack 10 eps |s| + 10 eps (test_cv.cpp:110-127).
"""
import numpy as np
import pytest

from paper_1102_2878_b200 import datagen

pytestmark = pytest.mark.gpu


def _naive_opts(dfgtb):
    return dfgtb.CvOptions(algorithm=dfgtb.Algorithm.naive)


def test_two_point_likelihood(dfgtb):
    h, d = 0.7, 0.9
    refs = np.array([[0.0], [d]])
    r = dfgtb.lkcv_score(refs, h, _naive_opts(dfgtb))
    assert r.score == pytest.approx(np.log(np.exp(-d * d / (2 * h * h)) / dfgtb.gaussian_normalizer(1, h)),
                                    rel=1e-12)
    assert r.clamped == 0


def test_two_point_least_squares_golden(dfgtb):
    h, d = 0.7, 0.9
    refs = np.array([[0.0], [d]])
    r = dfgtb.lscv_score(refs, h, _naive_opts(dfgtb))
    assert r.score == pytest.approx(-0.26698943846309625, rel=1e-12)
    # the same through the fused on-device CV path
    e = dfgtb.DualTreeEngine(refs, config=dfgtb.EngineConfig(epsilon=0.0))
    row = e.cv(h)
    assert row.ls_score == pytest.approx(-0.26698943846309625, rel=1e-12)


def test_device_cv_matches_host_formulas(dfgtb, orc):
    w = datagen.config(2, scale_n=0.1)
    e = dfgtb.DualTreeEngine(w.refs, config=dfgtb.EngineConfig(leaf_threshold=32))
    for s in (0.1, 1.0, 10.0):
        h = s * w.h_s
        s1, s2 = e.compute(None, h), e.compute(None, 2 * h)
        row = e.cv(h)
        lk, cl = orc.lkcv(2, h, s1)
        ls = orc.lscv(2, h, s1, 2 * h, s2)
        assert row.lk_score == pytest.approx(lk, rel=1e-12, abs=1e-12)
        assert row.lk_clamped == cl
        assert row.ls_score == pytest.approx(ls, rel=1e-10, abs=1e-14)


@pytest.mark.parametrize("h", [0.02, 0.1, 0.4])
def test_scores_agree_with_naive_within_slack(dfgtb, h):
    g = np.random.default_rng(14)
    refs = g.random((500, 2)) * 0.5 + 0.25 * (g.integers(0, 2, (500, 1)))
    eps = 0.01
    for kind in (dfgtb.CvScore.likelihood, dfgtb.CvScore.least_squares):
        fn = dfgtb.lkcv_score if kind is dfgtb.CvScore.likelihood else dfgtb.lscv_score
        naive = fn(refs, h, _naive_opts(dfgtb)).score
        fast = fn(refs, h, dfgtb.CvOptions(engine=dfgtb.EngineConfig(epsilon=eps))).score
        assert abs(fast - naive) <= 10 * eps * abs(naive) + 10 * eps


def test_sweep_rows_and_argmin(dfgtb, orc):
    w = datagen.config(2, scale_n=0.04)
    e = dfgtb.DualTreeEngine(w.refs, config=dfgtb.EngineConfig(leaf_threshold=32))
    rows = e.sweep(w.scales, w.h_s)
    assert [r.scale for r in rows] == list(w.scales)
    ls_naive, lk_naive = [], []
    for r in rows:
        ex = orc.naive_kde(w.refs, w.refs, r.h)
        ex2 = orc.naive_kde(w.refs, w.refs, 2 * r.h)
        ls_naive.append(orc.lscv(2, r.h, ex, 2 * r.h, ex2))
        lk_naive.append(orc.lkcv(2, r.h, ex)[0])
    assert int(np.argmin([r.ls_score for r in rows])) == int(np.argmin(ls_naive))
    with pytest.raises(ValueError):
        e.sweep([1.0, 0.5], w.h_s)
