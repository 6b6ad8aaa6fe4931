"""Synthetic BASELINE workloads: shapes, determinism, ranges (CPU)."""
import numpy as np
import pytest

from paper_1102_2878_b200 import datagen


@pytest.mark.parametrize("k,n,d", [(1, 10_000, 2), (2, 50_000, 2), (3, 200_000, 3), (4, 100_000, 5)])
def test_shapes_and_ranges(k, n, d):
    w = datagen.config(k, scale_n=0.05)
    assert w.refs.shape == (int(round(n * 0.05)), d)
    assert np.all(w.refs >= 0.0) and np.all(w.refs <= 1.0)
    assert w.h_s > 0 and w.queries is None
    w2 = datagen.config(k, scale_n=0.05)
    assert np.array_equal(w.refs, w2.refs)


def test_cfg2_clipping_hits_the_border():
    x = datagen.config(2).refs
    assert x.shape == (50_000, 2)
    # clipping puts points exactly on the unit-square border (zero-width boxes in
    # one dimension); exact duplicates for the nth_element fallback are exercised
    # by the quantized / duplicate fixtures in tests/golden/trees.npz instead
    assert ((x == 0.0) | (x == 1.0)).any(axis=1).sum() > 100


def test_cfg3_unit_cube_and_background():
    x = datagen.config(3, scale_n=0.1).refs
    assert np.allclose(x.min(axis=0), 0.0) and np.allclose(x.max(axis=0), 1.0)


def test_cfg5_fp32_widened():
    w = datagen.config(5, scale_n=0.002)
    assert w.queries is not None
    assert np.array_equal(w.refs, w.refs.astype(np.float32).astype(np.float64))
    assert np.array_equal(w.queries, w.queries.astype(np.float32).astype(np.float64))
    assert w.scales == (0.1, 1.0, 10.0)


def test_silverman():
    x = np.random.default_rng(0).random((1000, 2))
    s = np.mean(np.std(x, axis=0, ddof=1))
    assert datagen.silverman_h(x) == pytest.approx(1.06 * s * 1000 ** -0.2)


def test_sweep_scales():
    assert len(datagen.SWEEP_9) == 9 and datagen.SWEEP_9[4] == 1.0
    assert len(datagen.SWEEP_7) == 7
