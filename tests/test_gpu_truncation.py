"""The traversal's classification primitives on the GPU vs the reference, bit for bit.

The traversal (traverse.cu) evaluates the Lemma 3/4/5 bounds in a division-free form
and falls back to the reference's own expression near a tie, so its decisions must
be the reference's exactly -- an eps test cannot see a rewrite that picks a different
but still valid method, these tests can:
  * choose_best_method + the three least orders (truncation.cpp:85-166) on the 300
    committed reference decisions (tests/golden/truncation.json), on random tuples,
    and on tuples whose tau IS a reference bound value (exact ties);
  * box_distance_bounds_sq (kdtree.cpp:122-141) on the reference's goldens
    (test_kdtree.cpp:119-146) and bit-exact on random boxes.
"""
import ctypes as C
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gpu_choose(args):
    from paper_1102_2878_b200 import _capi
    a = np.ascontiguousarray(args, dtype=np.float64)
    out = np.zeros((a.shape[0], 5), np.int32)
    _capi.check(_capi.lib.dfgtb_choose_methods(a.shape[0], a.ctypes.data_as(C.POINTER(C.c_double)),
                                               out.ctypes.data_as(C.POINTER(C.c_int))))
    return out


def _gpu_box(d, boxes):
    from paper_1102_2878_b200 import _capi
    b = np.ascontiguousarray(boxes, dtype=np.float64)
    out = np.zeros((b.shape[0], 2))
    _capi.check(_capi.lib.dfgtb_box_bounds(b.shape[0], d, b.ctypes.data_as(C.POINTER(C.c_double)),
                                           out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


def _ref_orders(ref, nr, sq, sr, h, tau, pmax, d):
    """least_order over the reference's own bound functions (truncation.cpp:85-128)."""
    def least(bound, r, lim):
        if r >= lim:
            return 0
        for p in range(1, pmax + 1):
            if bound(nr, r, p, d) <= tau:
                return p
        return 0
    pf = least(ref.farfield_error_bound, sr / (2.0 * h), 1.0)
    pd = least(ref.farfield_error_bound, sq / (2.0 * h), 1.0)
    pt = least(ref.f2l_error_bound, max(sq, sr) / (4.0 * h), 0.5)
    return pf, pd, pt


def test_choose_on_committed_reference_decisions(dfgtb):
    rows = json.load(open(os.path.join(GOLD, "truncation.json")))
    out = _gpu_choose([r["args"] for r in rows])
    for r, o in zip(rows, out):
        assert (int(o[0]), int(o[1])) == (r["kind"], r["order"]), r["args"]


def _random_tuples(rng, n):
    d = rng.integers(1, 6, n)
    pmax = np.array([[8, 6, 4, 2, 2][k - 1] for k in d])
    pmax = np.where(rng.random(n) < 0.3, rng.integers(1, 9, n), pmax)
    nq, nr = rng.integers(1, 20000, n).astype(float), rng.integers(1, 20000, n).astype(float)
    sq, sr = rng.uniform(0, 0.4, n), rng.uniform(0, 0.4, n)
    h = 10 ** rng.uniform(-2.5, 0.5, n)
    tau = 10 ** rng.uniform(-4, 2, n) * nr
    cm = rng.integers(0, 2, n)
    return np.stack([nq, nr, sq, sr, h, tau, pmax, d, cm], axis=1)


def test_choose_and_orders_vs_reference_random(dfgtb, ref):
    rng = np.random.default_rng(2024)
    args = _random_tuples(rng, 4000)
    out = _gpu_choose(args)
    for a, o in zip(args, out):
        nq, nr, sq, sr, h, tau, pmax, d, cm = a
        kind, order = ref.choose_best_method(nq, nr, sq, sr, h, tau, int(pmax), int(d), int(cm))
        assert (int(o[0]), int(o[1])) == (kind, order), a
        assert tuple(int(v) for v in o[2:]) == _ref_orders(ref, nr, sq, sr, h, tau, int(pmax), int(d)), a


def test_choose_at_exact_ties(dfgtb, ref):
    """tau set to the reference's own bound at some order: the division-free fast test
    is within rounding of a tie there, and the decision must still be the reference's."""
    rng = np.random.default_rng(77)
    rows = []
    for _ in range(3000):
        d = int(rng.integers(1, 6))
        pmax = int(rng.integers(1, 9))
        nr = float(rng.integers(1, 5000))
        nq = float(rng.integers(1, 5000))
        h = 10 ** rng.uniform(-2, 0)
        sq, sr = rng.uniform(0, 0.9) * 2 * h, rng.uniform(0, 0.9) * 2 * h
        p = int(rng.integers(1, pmax + 1))
        which = int(rng.integers(0, 3))
        if which == 0:
            tau = ref.farfield_error_bound(nr, sr / (2.0 * h), p, d)
        elif which == 1:
            tau = ref.farfield_error_bound(nr, sq / (2.0 * h), p, d)
        else:
            r = max(sq, sr) / (4.0 * h)
            if r >= 0.5:
                continue
            tau = ref.f2l_error_bound(nr, r, p, d)
        if not np.isfinite(tau) or tau <= 0:
            continue
        # the tie itself and its two floating-point neighbours
        for t in (np.nextafter(tau, 0.0), tau, np.nextafter(tau, np.inf)):
            rows.append([nq, nr, sq, sr, h, t, pmax, d, int(rng.integers(0, 2))])
    args = np.array(rows)
    out = _gpu_choose(args)
    for a, o in zip(args, out):
        nq, nr, sq, sr, h, tau, pmax, d, cm = a
        kind, order = ref.choose_best_method(nq, nr, sq, sr, h, tau, int(pmax), int(d), int(cm))
        assert (int(o[0]), int(o[1])) == (kind, order), a
        assert tuple(int(v) for v in o[2:]) == _ref_orders(ref, nr, sq, sr, h, tau, int(pmax), int(d)), a


def test_box_bounds_reference_goldens(dfgtb):
    # test_kdtree.cpp:119-146
    g = _gpu_box(2, [[0, 0, 1, 1, 2, 0, 3, 1], [-1, 2, 1, 4, -1, 2, 1, 4], [1, 2, 1, 2, 4, 6, 4, 6]])
    assert np.sqrt(g[0, 0]) == pytest.approx(1.0, rel=1e-14)
    assert np.sqrt(g[0, 1]) == pytest.approx(3.1622776601683795, rel=1e-14)
    assert g[1, 0] == 0.0 and np.sqrt(g[1, 1]) == pytest.approx(np.sqrt(8.0), rel=1e-14)
    assert np.sqrt(g[2, 0]) == pytest.approx(5.0, rel=1e-14)
    assert np.sqrt(g[2, 1]) == pytest.approx(5.0, rel=1e-14)


@pytest.mark.parametrize("d", [1, 2, 3, 5, 8, 16])
def test_box_bounds_bit_exact_vs_reference(dfgtb, ref, d):
    rng = np.random.default_rng(300 + d)
    n = 2000
    lo_a = rng.normal(size=(n, d))
    lo_b = rng.normal(size=(n, d))
    # overlapping, nested, touching and point boxes
    ext_a = np.where(rng.random((n, d)) < 0.2, 0.0, rng.exponential(size=(n, d)))
    ext_b = np.where(rng.random((n, d)) < 0.2, 0.0, rng.exponential(size=(n, d)))
    boxes = np.concatenate([lo_a, lo_a + ext_a, lo_b, lo_b + ext_b], axis=1)
    got = _gpu_box(d, boxes)
    for i in range(n):
        want = ref.box_bounds_sq(boxes[i, :d], boxes[i, d:2 * d], boxes[i, 2 * d:3 * d],
                                 boxes[i, 3 * d:])
        assert got[i, 0] == want[0] and got[i, 1] == want[1], (d, i)
