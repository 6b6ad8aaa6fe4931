"""GPU DFGT sums vs the FP64 oracle: the per-query eps guarantee and the
reference's engine properties (test_engine.cpp, acceptance.cpp criterion 1).

Tolerance: |G_gpu - G_exact| <= eps * G_exact per query (the reference's contract,
engine.hpp:93), checked with a 1e-12 relative slack for FP64 summation order.
"""
import numpy as np
import pytest

from paper_1102_2878_b200 import datagen

pytestmark = pytest.mark.gpu
SLACK = 1e-12


def _mixture(n, d, seed):
    g = np.random.default_rng(seed)
    c = g.random((6, d))
    comp = g.integers(0, 6, n)
    return c[comp] + 0.05 * g.standard_normal((n, d))


def _check(approx, exact, eps):
    ok = exact > 0
    rel = np.abs(approx[ok] - exact[ok]) / exact[ok]
    assert rel.max(initial=0.0) <= eps * (1 + 1e-9) + SLACK, rel.max()
    return rel.max(initial=0.0)


def test_single_point_is_one(dfgtb):
    p = np.array([[0.3, -0.7]])
    assert dfgtb.dfgt_kde(p, p, 0.8).tolist() == [1.0]
    assert dfgtb.dfd_kde(p, p, 0.8, 0.01).tolist() == [1.0]


def test_naive_goldens(dfgtb, orc):
    p = np.array([[1.0, 2.0]])
    assert dfgtb.naive_kde(p, p, 0.5).tolist() == [1.0]
    s = dfgtb.naive_kde(np.array([[0.0]]), np.array([[0.0], [3.0]]), 1.5)
    assert s[0] == pytest.approx(1.0 + np.exp(-9.0 / (2 * 1.5 * 1.5)), rel=1e-14)
    x = np.random.default_rng(1).random((700, 3))
    assert np.allclose(dfgtb.naive_kde(x, x, 0.07), orc.naive_kde(x, x, 0.07), rtol=1e-13, atol=0)


def test_dimension_mismatch_raises(dfgtb):
    with pytest.raises(ValueError):
        dfgtb.naive_kde(np.zeros((1, 2)), np.zeros((1, 3)), 1.0)
    with pytest.raises(ValueError):
        dfgtb.dfgt_kde(np.zeros((1, 2)), np.zeros((1, 3)), 1.0)


def test_invalid_arguments(dfgtb):
    x = np.random.default_rng(0).random((50, 2))
    with pytest.raises(ValueError):
        dfgtb.DualTreeEngine(x, config=dfgtb.EngineConfig(epsilon=-1.0))
    with pytest.raises(ValueError):
        dfgtb.DualTreeEngine(x, config=dfgtb.EngineConfig(leaf_threshold=0))
    with pytest.raises(ValueError):
        dfgtb.DualTreeEngine(x, config=dfgtb.EngineConfig(p_max=16))
    e = dfgtb.DualTreeEngine(x)
    with pytest.raises(ValueError):
        e.compute(None, 0.0)
    with pytest.raises(ValueError):
        e.compute(None, -1.0)


def test_dfd_zero_tolerance_matches_naive(dfgtb, orc):
    pts = _mixture(300, 2, 9)
    exact = orc.naive_kde(pts, pts, 0.05)
    approx = dfgtb.dfd_kde(pts, pts, 0.05, 0.0, 8)
    assert dfgtb.verify_relative_error(approx, exact).max_relative_error <= 1e-12


@pytest.mark.parametrize("h", [0.001, 0.05, 0.5, 5.0])
def test_dfd_contract(dfgtb, orc, h):
    pts = _mixture(1000, 2, 12)
    _check(dfgtb.dfd_kde(pts, pts, h, 0.01), orc.naive_kde(pts, pts, h), 0.01)


def test_dfgt_contract_across_scales(dfgtb, orc):
    pts = _mixture(500, 2, 21)
    e = dfgtb.DualTreeEngine(pts, dfgtb.Mode.series, dfgtb.EngineConfig(epsilon=0.01))
    for scale in (1e-3, 1e-2, 1e-1, 1.0, 10.0, 100.0, 1000.0):
        h = scale * 0.05
        _check(e.compute(None, h), orc.naive_kde(pts, pts, h), 0.01)


def test_separate_query_and_reference(dfgtb, orc):
    refs = _mixture(700, 3, 31)
    q = np.random.default_rng(32).random((350, 3))
    for h in (0.05, 0.2, 2.0):
        approx = dfgtb.dfgt_kde(q, refs, h, dfgtb.EngineConfig(epsilon=0.001))
        _check(approx, orc.naive_kde(q, refs, h), 0.001)


def test_global_guarantee_random_instances(dfgtb, orc):
    rng = np.random.default_rng(123)
    for inst in range(15):
        d = 1 + inst % 3
        n = 200 + 50 * inst
        pts = _mixture(n, d, 400 + inst)
        h = 10 ** rng.uniform(-3, 3)
        exact = orc.naive_kde(pts, pts, h)
        for eps in (0.1, 0.01, 0.001):
            _check(dfgtb.dfgt_kde(pts, pts, h, dfgtb.EngineConfig(epsilon=eps)), exact, eps)


def test_term_count_cost_model(dfgtb, orc):
    pts = _mixture(400, 2, 77)
    cfg = dfgtb.EngineConfig(epsilon=0.01, cost_model=dfgtb.CostModel.term_count)
    for h in (0.02, 0.2, 2.0):
        _check(dfgtb.dfgt_kde(pts, pts, h, cfg), orc.naive_kde(pts, pts, h), 0.01)


def test_loose_tolerance_single_prune(dfgtb):
    pts = _mixture(150, 2, 5)
    e = dfgtb.DualTreeEngine(pts, dfgtb.Mode.series,
                             dfgtb.EngineConfig(epsilon=1e6, leaf_threshold=10))
    s = e.compute(None, 1.0)
    assert e.last_stats().pairs_visited == 1
    assert np.all(np.isfinite(s))


def test_bit_identical_runs(dfgtb):
    pts = _mixture(800, 2, 55)
    a = dfgtb.dfgt_kde(pts, pts, 0.02)
    b = dfgtb.dfgt_kde(pts, pts, 0.02)
    assert np.array_equal(a, b)
    w = datagen.config(2, scale_n=0.2)
    e = dfgtb.DualTreeEngine(w.refs, config=dfgtb.EngineConfig(leaf_threshold=32))
    for h in (w.h_s, 3 * w.h_s):
        assert np.array_equal(e.compute(None, h), e.compute(None, h))


def test_kernel_evals_monotone_in_eps(dfgtb):
    pts = _mixture(1000, 2, 66)
    prev = None
    for eps in (1e-3, 1e-2, 1e-1):
        e = dfgtb.DualTreeEngine(pts, config=dfgtb.EngineConfig(epsilon=eps))
        e.compute(None, 0.05)
        ev = e.last_stats().kernel_evaluations
        assert prev is None or ev <= prev
        prev = ev


def test_series_prunes_engage(dfgtb):
    pts = _mixture(2000, 2, 99)
    e = dfgtb.DualTreeEngine(pts, config=dfgtb.EngineConfig(epsilon=0.01))
    e.compute(None, 0.1)
    st = e.last_stats()
    assert st.prunes_farfield + st.prunes_direct_local + st.prunes_far_to_local > 0


def test_all_duplicates_exact(dfgtb):
    pts = np.tile([[0.25, -1.5]], (64, 1))
    e = dfgtb.DualTreeEngine(pts, config=dfgtb.EngineConfig(epsilon=0.0, leaf_threshold=4))
    assert np.all(e.compute(None, 0.7) == 64.0)


def test_six_dimensional_order_one(dfgtb, orc):
    pts = _mixture(300, 6, 11)
    e = dfgtb.DualTreeEngine(pts, config=dfgtb.EngineConfig(epsilon=0.01))
    assert e.p_max() == 1
    for h in (0.05, 0.5, 5.0):
        _check(e.compute(None, h), orc.naive_kde(pts, pts, h), 0.01)


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_config_generators_small(dfgtb, orc, k):
    """Every config's distribution at reduced N, full eps check vs the CPU oracle
    (acceptance.cpp criterion 1 analogue)."""
    w = datagen.config(k, scale_n=0.05 if k != 1 else 0.3)
    for eps in w.epsilons:
        e = dfgtb.DualTreeEngine(w.refs, config=dfgtb.EngineConfig(epsilon=eps, leaf_threshold=32,
                                                                    p_max=w.p_max or None))
        for s in (w.scales if len(w.scales) > 1 else (0.5, 1.0, 2.0)):
            h = s * w.h_s
            exact = orc.naive_kde(w.refs, w.refs, h)
            _check(e.compute(None, h), exact, eps)


def test_dfgt_matches_reference_within_eps(dfgtb, ref):
    """GPU vs the compiled reference DFGT: both within eps of exact, so within
    2 eps of each other; prune decisions differ (BFS vs DFS order)."""
    w = datagen.config(2, scale_n=0.05)
    re = ref.engine(w.refs, eps=0.01, leaf=32)
    e = dfgtb.DualTreeEngine(w.refs, config=dfgtb.EngineConfig(leaf_threshold=32))
    for s in w.scales:
        h = s * w.h_s
        a = e.compute(None, h)
        b, _ = re.compute(h)
        assert np.all(np.abs(a - b) <= 0.0201 * np.abs(b) + 1e-300)


def test_batched_bandwidths_bit_identical_to_single(dfgtb):
    """compute_batch runs every bandwidth through one lock-step traversal; each slot's
    decisions and accumulation order are its own, so results equal one-at-a-time runs
    bit for bit (Q = R and Q != R)."""
    w = datagen.config(2, scale_n=0.05)
    e = dfgtb.DualTreeEngine(w.refs, config=dfgtb.EngineConfig(leaf_threshold=32))
    hs = [s * w.h_s for s in w.scales] + [2 * s * w.h_s for s in w.scales]
    batch = e.compute_batch(None, hs)
    bstats = e.batch_stats()
    for b, h in enumerate(hs):
        single = e.compute(None, h)
        assert np.array_equal(batch[b], single), b
        a, s = vars(bstats[b]), vars(e.last_stats())
        a.pop("levels"), s.pop("levels")  # a batch runs until its deepest slot is done
        assert a == s
    q = np.random.default_rng(8).random((777, 2))
    batch = e.compute_batch(q, hs[:5])
    for b, h in enumerate(hs[:5]):
        assert np.array_equal(batch[b], e.compute(q, h))


def test_l2l_chain_matches_direct_ancestor_evaluation(dfgtb, orc):
    """local_pushdown=1 runs the reference's L2L push-down chain (post_process,
    engine.cpp:294-304); the default evaluates every ancestor's local expansion at
    the query.  Exact polynomial re-centring: both agree to rounding."""
    w = datagen.config(2, scale_n=0.04)
    for s in (0.3, 1.0, 3.0, 10.0):
        h = s * w.h_s
        a = dfgtb.DualTreeEngine(w.refs, config=dfgtb.EngineConfig(leaf_threshold=32)).compute(None, h)
        e = dfgtb.DualTreeEngine(w.refs, config=dfgtb.EngineConfig(leaf_threshold=32, local_pushdown=1))
        b = e.compute(None, h)
        assert np.max(np.abs(a - b) / np.abs(b)) <= 1e-10
        _check(b, orc.naive_kde(w.refs, w.refs, h), 0.01)


def test_fast_exp_accuracy(dfgtb, orc):
    """The base case's table-driven exp(-y) vs libm: eps = 0 base-case-only sums agree
    with the exact oracle to summation-order rounding, including pairs deep in the
    underflow range (careful path)."""
    g = np.random.default_rng(3)
    x = g.random((600, 2)) * np.array([1.0, 0.01])
    for h in (0.002, 0.01, 0.05, 0.3):
        approx = dfgtb.dfd_kde(x, x, h, 0.0, 16)
        exact = orc.naive_kde(x, x, h)
        assert np.max(np.abs(approx - exact) / exact) <= 1e-13


@pytest.mark.parametrize("d,leaf", [(1, 700), (2, 16), (2, 300), (3, 7), (3, 200), (4, 50), (5, 90)])
def test_base_case_tiles_exact(dfgtb, orc, d, leaf):
    """eps = 0: every pair goes through the base case.  Leaves larger than the
    shared-memory stream tile (chunked staging), every query-group remainder, and
    Q != R, all to summation-order rounding of the exact sums."""
    g = np.random.default_rng(10 + d)
    r = g.random((900, d))
    q = g.random((333, d))
    for h in (0.03, 0.2, 2.0):
        for qq in (r, q):
            approx = dfgtb.dfd_kde(qq, r, h, 0.0, leaf)
            exact = orc.naive_kde(qq, r, h)
            assert np.max(np.abs(approx - exact) / exact) <= 1e-13


def test_mufu_exp_error_within_charge(dfgtb):
    """The base case's MUFU exp (eps >= 1e-4): exhaustive max relative error over every
    fixed-point argument (and the clamp beyond z = 1021), plus the fixed-point rounding
    bound (D + 2) ln2 2^-21 at D = 5, stays below the 4e-6 the traversal charges."""
    from paper_1102_2878_b200 import _capi
    err = _capi.lib.dfgtb_mufu_exp_error()
    assert 0.0 <= err < 1e-6
    assert err + 7 * np.log(2.0) * 2.0 ** -21 < 4e-6


@pytest.mark.parametrize("k", [2, 3, 4])
def test_mufu_path_meets_eps(dfgtb, orc, k):
    """eps = 0.01 runs the MUFU base case: per-query error within eps of the exact
    sums at every sweep scale, and within 1e-5 of the FP64-exp engine's sums."""
    import os
    w = datagen.config(k, scale_n=0.03)
    for s in w.scales:
        h = s * w.h_s
        got = dfgtb.dfgt_kde(w.refs, w.refs, h, dfgtb.EngineConfig(epsilon=0.01, leaf_threshold=32))
        _check(got, orc.naive_kde(w.refs, w.refs, h), 0.01)


def test_base_exp_mode_selection(dfgtb, orc, monkeypatch):
    """eps >= 1e-4 runs the MUFU base case (charged), smaller eps or DFGTB_EXACT_EXP the
    FP64 exp; both meet eps, and the MUFU self term is exactly K(0) = 1 (Q = R leave-
    one-out sums G - 1 agree with the FP64 engine where they are well above eps G)."""
    from paper_1102_2878_b200 import _capi
    w = datagen.config(2, scale_n=0.04)
    h = w.h_s
    with dfgtb.DualTreeEngine(w.refs, config=dfgtb.EngineConfig(epsilon=0.01, leaf_threshold=32)) as e:
        assert _capi.lib.dfgtb_base_exp_mode(e.handle) == 2  # FP32 leaf pairs, MUFU-FP64 rest
        fast = e.compute(None, h)
    with dfgtb.DualTreeEngine(w.refs, config=dfgtb.EngineConfig(epsilon=1e-3, leaf_threshold=32)) as e:
        assert _capi.lib.dfgtb_base_exp_mode(e.handle) == 1
    with dfgtb.DualTreeEngine(w.refs, config=dfgtb.EngineConfig(epsilon=1e-5, leaf_threshold=32)) as e:
        assert _capi.lib.dfgtb_base_exp_mode(e.handle) == 0
    monkeypatch.setenv("DFGTB_EXACT_EXP", "1")
    with dfgtb.DualTreeEngine(w.refs, config=dfgtb.EngineConfig(epsilon=0.01, leaf_threshold=32)) as e:
        assert _capi.lib.dfgtb_base_exp_mode(e.handle) == 0
        exact_path = e.compute(None, h)
    exact = orc.naive_kde(w.refs, w.refs, h)
    _check(fast, exact, 0.01)
    _check(exact_path, exact, 0.01)
    # tiny bandwidth: every query's sum is its self term plus a tiny rest
    tiny = 1e-3 * w.h_s
    monkeypatch.delenv("DFGTB_EXACT_EXP")
    with dfgtb.DualTreeEngine(w.refs, config=dfgtb.EngineConfig(epsilon=0.01, leaf_threshold=32)) as e:
        assert _capi.lib.dfgtb_base_exp_mode(e.handle) == 2
        g = e.compute(None, tiny)
    ex = orc.naive_kde(w.refs, w.refs, tiny)
    assert np.all(g >= 1.0) and np.max(np.abs((g - 1.0) - (ex - 1.0))) <= 0.01 * np.max(ex)


def test_float32_inputs_match_widened(dfgtb):
    """Config 5's fp32 inputs: dfgtb_create_f32 / dfgtb_compute_batch_f32 widen exactly
    on the device, so results are bit-identical to the float64 path on the same values."""
    w = datagen.config(5, scale_n=0.002)
    r32, q32 = w.refs.astype(np.float32), w.queries.astype(np.float32)
    hs = [s * w.h_s for s in w.scales]
    cfg = dfgtb.EngineConfig(epsilon=0.01, leaf_threshold=32)
    with dfgtb.DualTreeEngine(r32, config=cfg) as e32:
        a = e32.compute_batch(q32, hs)
    with dfgtb.DualTreeEngine(r32.astype(np.float64), config=cfg) as e64:
        b = e64.compute_batch(q32.astype(np.float64), hs)
    assert np.array_equal(a, b)


def test_compute_batch_into_out(dfgtb):
    """compute_batch(..., out=) writes the same sums into a caller's (e.g. pinned) buffer,
    for float64 and float32 queries, and rejects a wrongly shaped one."""
    g = np.random.default_rng(12)
    r, q = g.random((3000, 3)), g.random((1000, 3))
    hs = [0.02, 0.05, 0.2]
    with dfgtb.DualTreeEngine(r, config=dfgtb.EngineConfig(epsilon=0.01, leaf_threshold=32)) as e:
        for qq in (q, q.astype(np.float32)):
            want = e.compute_batch(qq, hs)
            out = np.full((3, 1000), -1.0)
            got = e.compute_batch(qq, hs, out=out)
            assert got is out and np.array_equal(out, want)
        with pytest.raises(ValueError):
            e.compute_batch(q, hs, out=np.empty((2, 1000)))
