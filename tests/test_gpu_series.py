"""GPU series primitives (the device functions the traversal kernels use) vs the
oracle restatement of series.cpp, on random inputs, reference table layout.

Tolerance 1e-12 relative to the table's scale (the reference's own exactness bar
for F2F is 1e-12 and for L2L 1e-9, acceptance.cpp:298-305, 330-340); the GPU
builds monomials from power tables instead of the ancestor recurrence, so results
agree to rounding, not bit for bit.
"""
import ctypes as C

import numpy as np
import pytest

from paper_1102_2878_b200 import _capi

pytestmark = pytest.mark.gpu
_D = C.POINTER(C.c_double)


def op(k, d, p, inp, n, a, b, h, order, out):
    inp = np.ascontiguousarray(inp, dtype=np.float64)
    out = np.ascontiguousarray(out, dtype=np.float64).copy()
    a = np.ascontiguousarray(a, dtype=np.float64)
    bb = np.ascontiguousarray(b if b is not None else a, dtype=np.float64)
    _capi.check(_capi.lib.dfgtb_series_op(k, d, p, inp.ctypes.data_as(_D), n, a.ctypes.data_as(_D),
                                          bb.ctypes.data_as(_D), h, order, out.ctypes.data_as(_D)))
    return out


def close(a, b, tol=1e-12):
    scale = max(1.0, float(np.max(np.abs(b))))
    assert np.max(np.abs(np.asarray(a) - np.asarray(b))) <= tol * scale


CASES = [(1, 8), (2, 6), (3, 4), (4, 2), (5, 2), (2, 3), (3, 2)]


@pytest.mark.parametrize("d,p", CASES)
def test_series_primitives(orc, d, p):
    rng = np.random.default_rng(10 * d + p)
    h = 0.3
    T = p ** d
    c = rng.random(d)
    pts = c + 0.2 * (rng.random((17, d)) - 0.5)
    M_o = orc.moments(p, pts, c, h)
    M_g = op(0, d, p, pts, len(pts), c, None, h, 0, np.zeros(T))
    close(M_g, M_o)
    q = c + 0.9 * rng.random(d)
    for order in range(1, p + 1):
        close([op(1, d, p, M_o, 0, c, q, h, order, np.zeros(1))[0]],
              [orc.eval_farfield(p, M_o, c, q, h, order)])
        qc = q + 0.05
        L0 = rng.random(T)
        close(op(2, d, p, pts, len(pts), qc, None, h, order, L0),
              orc.direct_local(p, pts, qc, h, order, L0))
        close(op(3, d, p, M_o, 0, c, qc, h, order, L0), orc.f2l(p, M_o, c, qc, h, order, L0))
        c2 = qc + 0.03 * rng.random(d)
        close(op(4, d, p, L0, 0, qc, c2, h, order, np.zeros(T)),
              orc.l2l(p, L0, qc, c2, h, order), tol=1e-11)
        close([op(5, d, p, L0, 0, qc, q, h, order, np.zeros(1))[0]],
              [orc.eval_local(p, L0, qc, q, h, order)])


def test_series_goldens():
    # test_series.cpp:118-130: h_1(1) = 2 e^-1 = 0.7357588823428847 (via eval_farfield
    # of a unit order-2 table: M = e_1 selects h_1 along the single dimension)
    T = 2
    M = np.array([0.0, 1.0])
    h = 1.0 / np.sqrt(2.0)  # scaled argument (q - c)/(h sqrt 2) = q - c
    v = op(1, 1, 2, M, 0, np.zeros(1), np.ones(1), h, 2, np.zeros(1))[0]
    assert v == pytest.approx(0.7357588823428847, rel=1e-14)
    assert T == 2
