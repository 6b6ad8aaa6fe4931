"""The FP32 base case (leaf pairs flagged with order bit 2, eps >= 5e-3): FP32 differences,
ex2.approx.ftz.f32 of the whole argument shifted by S = 64 (terms 2^(S - z), scaled back
by 2^-S per tile in FP64), FP32 partial sums, Q = R self pairs masked and K(0) = 1 added
exactly.  Its per-term relative
error must stay below kF32Charge = 2e-4, the share of eps the traversal pays for it
(derivation at execute.cu FPt), and the engine must still meet eps per query.
"""
import numpy as np
import pytest

from paper_1102_2878_b200 import datagen

pytestmark = pytest.mark.gpu
F32_CHARGE = 2e-4
U = 2.0 ** -24


def _terms(d, q, r, c):
    from paper_1102_2878_b200 import _capi
    D = _capi._D
    q = np.ascontiguousarray(q, dtype=np.float64)
    r = np.ascontiguousarray(r, dtype=np.float64)
    c = np.ascontiguousarray(c, dtype=np.float64)
    out = np.empty(len(q))
    _capi.check(_capi.lib.dfgtb_f32_terms(d, q.ctypes.data_as(D), r.ctypes.data_as(D), c.ctypes.data_as(D),
                                          len(q), out.ctypes.data_as(D)))
    return out


def test_f32_exp_error_exhaustive():
    """ex2.approx.ftz.f32 over every FP32 argument in [-126, S = 64] (and 2^S exact)."""
    from paper_1102_2878_b200 import _capi
    err = _capi.lib.dfgtb_f32_exp_error()
    assert 0.0 <= err < 2.0 ** -21
    # the charge covers the exp, the distance bound at D = 5 (coordinate rounding
    # 2 sqrt(z) u (150 + sqrt z), differences 2 z u, sums D z u at z = 127) and the FP32
    # partial sums (21 roundings: <= 16 terms per lane per 512-point tile + 5 warp levels)
    z = 127.0
    dz = 2 * np.sqrt(z) * (150 + np.sqrt(z)) * U + 2 * z * U + 5 * z * U
    assert abs(dz - 2.697e-4) < 1e-6
    assert err + dz * np.log(2.0) + 21 * U < F32_CHARGE


@pytest.mark.parametrize("d", [1, 2, 3, 4, 5])
def test_f32_terms_within_charge(d):
    """Pairs at the extremes the traversal allows: queries up to 75 units from the
    centre (half the query leaf's diagonal bound), references at any distance with z <= 125
    (terms >= 2^-125, no flush), the reference on the far side of the centre (largest
    |r|), large centre offsets; against 2^-z in FP64."""
    g = np.random.default_rng(100 + d)
    n = 200000
    c = g.uniform(-300.0, 300.0, d)
    u = g.standard_normal((n, d))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    rad = np.where(g.random(n) < 0.5, 75.0, 75.0 * g.random(n) ** (1.0 / d))
    q = c + u * rad[:, None]
    v = g.standard_normal((n, d))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    far = g.random(n) < 0.3
    v[far] = -u[far]  # reference beyond the centre: |r - c| = |q - c| + sqrt(z)
    z = np.where(g.random(n) < 0.2, 125.0 * g.random(n) ** 0.25, 125.0 * g.random(n))
    r = q + v * np.sqrt(z)[:, None]
    want = np.exp2(-np.sum((q - r) ** 2, axis=1))
    got = _terms(d, q, r, c)
    rel = np.abs(got - want) / want
    assert rel.max() < F32_CHARGE - 21 * U, rel.max()
    # the self pair (q = r) is exactly 2^-0 = 1
    got0 = _terms(d, q[:1000], q[:1000], c)
    assert np.all(got0 == 1.0)


def test_f32_far_terms_flush_to_zero():
    """Terms with z >= 191 (below 2^-190) are 0 or below 2^-189: dropped mass only."""
    g = np.random.default_rng(7)
    d, n = 3, 10000
    c = np.zeros(d)
    q = g.uniform(-43.0, 43.0, (n, d))
    v = g.standard_normal((n, d))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    z = 191.0 + g.exponential(2000.0, n)
    r = q + v * np.sqrt(z)[:, None]
    got = _terms(d, q, r, c)
    assert np.all(got < 2.0 ** -189)


def test_f32_shift_keeps_small_terms():
    """127 < z <= 185: terms below FP32's normal range survive (the shift), with a
    relative error of at most ~2.6e-4 (the derivation's terms at z = 185; they weigh
    <= |R| 2^-127 against G >= 1e-20, so the charge still holds)."""
    g = np.random.default_rng(8)
    d, n = 2, 20000
    c = np.zeros(d)
    u = g.standard_normal((n, d))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    q = c + u * 75.0 * g.random(n)[:, None]
    v = g.standard_normal((n, d))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    z = 127.0 + 58.0 * g.random(n)
    r = q + v * np.sqrt(z)[:, None]
    want = np.exp2(-np.sum((q - r) ** 2, axis=1))
    got = _terms(d, q, r, c)
    zz = 185.0
    bound = (2 * np.sqrt(zz) * (150 + np.sqrt(zz)) + 2 * zz + d * zz) * U * np.log(2.0) + 2.0 ** -21
    assert np.all(got > 0)
    assert np.max(np.abs(got - want) / want) < bound


@pytest.mark.parametrize("k", [2, 3, 5])
def test_f32_path_meets_eps_and_is_used(dfgtb, orc, k, monkeypatch):
    """eps = 0.01 sums with the FP32 base case are within eps of the exact sums at every
    sweep scale, and the FP32 kernel ran tasks (dfgtb_last_base_split); with
    DFGTB_NO_F32 every task runs on the FP64 kernel."""
    import ctypes
    from paper_1102_2878_b200 import _capi
    w = datagen.config(k, scale_n=0.03 if k != 5 else 0.004)
    q = w.refs if w.queries is None else w.queries
    cfg = dfgtb.EngineConfig(epsilon=0.01, leaf_threshold=32)
    a, b = ctypes.c_int(), ctypes.c_int()
    nf32 = 0
    with dfgtb.DualTreeEngine(w.refs, config=cfg) as e:
        for s in w.scales:
            h = s * w.h_s
            got = e.compute(None if w.queries is None else q, h)
            _capi.check(_capi.lib.dfgtb_last_base_split(e.handle, ctypes.byref(a), ctypes.byref(b), None, None))
            nf32 += a.value
            exact = orc.naive_kde(q, w.refs, h)
            ok = exact > 0
            rel = np.abs(got[ok] - exact[ok]) / exact[ok]
            assert rel.max() <= 0.01, (s, rel.max())
    assert nf32 > 0
    monkeypatch.setenv("DFGTB_NO_F32", "1")
    with dfgtb.DualTreeEngine(w.refs, config=cfg) as e:
        e.compute(None if w.queries is None else q, w.h_s)
        _capi.check(_capi.lib.dfgtb_last_base_split(e.handle, ctypes.byref(a), ctypes.byref(b), None, None))
        assert a.value == 0 and b.value > 0


def test_f32_self_term_exact(dfgtb, orc, monkeypatch):
    """Q = R where the FP32 path applies: the self pair is masked out of the FP32 sums and
    K(0) = 1 added exactly, so G >= 1, an isolated point keeps G = 1 exactly, and every
    sum is within eps of the exact one."""
    g = np.random.default_rng(3)
    x = np.vstack([g.random((3000, 2)) * 0.1, [[5.0, 5.0], [5.3, 5.0], [9.0, 9.0]]])
    cfg = dfgtb.EngineConfig(epsilon=0.01, leaf_threshold=32)
    for h in (0.003, 0.01, 0.05):
        got = dfgtb.dfgt_kde(x, x, h, cfg)
        monkeypatch.setenv("DFGTB_NO_F32", "1")
        ref = dfgtb.dfgt_kde(x, x, h, cfg)
        monkeypatch.delenv("DFGTB_NO_F32")
        exact = orc.naive_kde(x, x, h)
        assert np.all(got >= 1.0 - 1e-6)
        assert got[-1] == 1.0
        assert np.max(np.abs(got - exact) / exact) <= 0.01
