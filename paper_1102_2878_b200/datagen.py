"""Seeded synthetic workloads for the five BASELINE.json configs.

BASELINE names no public dataset (the paper's datasets are not available), so these
generators stand in with the stated shapes, sizes and distributions.  The same bytes
feed the GPU engine and the CPU reference.  Seeds: config k uses 1000 + k; config 5's
reference set uses 2005.  numpy's PCG64 `Generator` is the bit source.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

SWEEP_9 = tuple(10.0 ** k for k in (-3, -2, -1, -0.5, 0, 0.5, 1, 2, 3))
SWEEP_7 = tuple(10.0 ** k for k in (-2, -1, -0.5, 0, 0.5, 1, 2))


def silverman_h(x: np.ndarray) -> float:
    """h_s = 1.06 * sigma_bar * N^(-1/5), sigma_bar = mean per-dim sample std (n-1)."""
    n = x.shape[0]
    sigma = float(np.mean(np.std(x, axis=0, ddof=1)))
    return 1.06 * sigma * n ** (-0.2)


def uniform(n: int, d: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).random((n, d))


def gauss_mixture_2d(n: int, seed: int, k: int = 16) -> np.ndarray:
    """Config 2: k isotropic Gaussians, centres U[0,1]^2, std log-U[.005,.05], equal
    weights, clipped to [0,1]^2 (clipping creates exact duplicates on the border)."""
    g = np.random.default_rng(seed)
    centres = g.random((k, 2))
    sig = np.exp(g.uniform(np.log(0.005), np.log(0.05), size=k))
    comp = g.integers(0, k, size=n)
    x = centres[comp] + sig[comp, None] * g.standard_normal((n, 2))
    return np.clip(x, 0.0, 1.0)


def _haar_rotation(g: np.random.Generator, d: int) -> np.ndarray:
    a = g.standard_normal((d, d))
    q, r = np.linalg.qr(a)
    return q * np.sign(np.diag(r))[None, :]


def clustered_3d(n: int, seed: int, k: int = 64, background: float = 0.10) -> np.ndarray:
    """Config 3: k rotated anisotropic Gaussian clusters (axis stds log-U[.002,.08]),
    sizes ~ j^-1.5, plus a uniform background over the clusters' bounding box, then
    min-max rescaled per dimension to the unit cube."""
    g = np.random.default_rng(seed)
    n_bg = int(round(background * n))
    n_cl = n - n_bg
    w = np.arange(1, k + 1, dtype=np.float64) ** -1.5
    w /= w.sum()
    sizes = g.multinomial(n_cl, w)
    centres = g.random((k, 3))
    parts = []
    for j in range(k):
        rot = _haar_rotation(g, 3)
        std = np.exp(g.uniform(np.log(0.002), np.log(0.08), size=3))
        z = g.standard_normal((sizes[j], 3)) * std[None, :]
        parts.append(centres[j] + z @ rot.T)
    cl = np.concatenate(parts, axis=0)
    lo, hi = cl.min(axis=0), cl.max(axis=0)
    bg = lo + (hi - lo) * g.random((n_bg, 3))
    x = np.concatenate([cl, bg], axis=0)
    x = x[g.permutation(n)]
    lo, hi = x.min(axis=0), x.max(axis=0)
    return (x - lo) / (hi - lo)


def full_cov_mixture_5d(n: int, seed: int, k: int = 8) -> np.ndarray:
    """Config 4: k Gaussians with Sigma = A A^T + 0.01 I, A_ij ~ N(0, 0.1^2), means
    U[0,1]^5, equal weights; rescaled to the unit hypercube."""
    g = np.random.default_rng(seed)
    d = 5
    means = g.random((k, d))
    chols = []
    for _ in range(k):
        a = 0.1 * g.standard_normal((d, d))
        chols.append(np.linalg.cholesky(a @ a.T + 0.01 * np.eye(d)))
    comp = g.integers(0, k, size=n)
    z = g.standard_normal((n, d))
    x = np.empty((n, d))
    for j in range(k):
        m = comp == j
        x[m] = means[j] + z[m] @ chols[j].T
    lo, hi = x.min(axis=0), x.max(axis=0)
    return (x - lo) / (hi - lo)


@dataclass
class Workload:
    name: str
    refs: np.ndarray
    queries: np.ndarray | None          # None -> Q = R
    h_s: float
    scales: tuple = field(default_factory=tuple)
    epsilons: tuple = (0.01,)
    leaf: int = 32
    p_max: int = 0                      # 0 -> reference default
    scores: tuple = ("lk", "ls")


def config(k: int, scale_n: float = 1.0) -> Workload:
    """BASELINE.json configs[k-1]; scale_n < 1 shrinks N for parity tests."""
    def N(n):
        return max(2, int(round(n * scale_n)))
    if k == 1:
        x = uniform(N(10_000), 2, 1001)
        return Workload("cfg1_uniform2d_10k", x, None, silverman_h(x), (1.0,), scores=("lk", "ls"))
    if k == 2:
        x = gauss_mixture_2d(N(50_000), 1002)
        return Workload("cfg2_mix16_2d_50k", x, None, silverman_h(x), SWEEP_9, scores=("lk", "ls"))
    if k == 3:
        x = clustered_3d(N(200_000), 1003)
        return Workload("cfg3_clustered3d_200k", x, None, silverman_h(x), SWEEP_9, scores=("ls",))
    if k == 4:
        x = full_cov_mixture_5d(N(100_000), 1004)
        return Workload("cfg4_mix8_5d_100k", x, None, silverman_h(x), SWEEP_7,
                        epsilons=(0.01, 0.001), scores=("lk",))
    if k == 5:
        r = clustered_3d(N(1_000_000), 2005).astype(np.float32).astype(np.float64)
        q = uniform(N(1_000_000), 3, 1005).astype(np.float32).astype(np.float64)
        return Workload("cfg5_R1M_Q1M_3d", r, q, silverman_h(r), (0.1, 1.0, 10.0), scores=())
    raise ValueError(f"unknown config {k}")
