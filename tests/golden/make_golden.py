#!/usr/bin/env python
"""Generate the committed golden fixtures from the REFERENCE itself.

Runs the unmodified reference compiled from /root/reference (oracle/_ref/
libdfgt_ref.so, see oracle/Makefile) on small seeded inputs and stores inputs and
outputs here, so the GPU box (where /root/reference does not exist) can check
parity against the reference's own results:

  trees.npz       KdTree::build arrays (kdtree.cpp:21-109) for 8 datasets
  sums.npz        DualTreeEngine::compute sums + TraversalStats, naive_kde sums
  cv.json         lkcv_from_sums / lscv_from_sums on those sums
  series.npz      series primitives (series.cpp) on random inputs
  truncation.json error bounds + choose_best_method (truncation.cpp)

  python tests/golden/make_golden.py      (needs oracle/_ref; run in the build container)
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import load_reference  # noqa: E402
from paper_1102_2878_b200 import datagen  # noqa: E402


def datasets():
    g = np.random.default_rng(77)
    out = {
        "uniform2d": (datagen.uniform(1200, 2, 11), 32),
        "mix2d_clipped": (datagen.gauss_mixture_2d(2000, 12), 32),
        "clustered3d": (datagen.clustered_3d(1500, 13), 16),
        "mix5d": (datagen.full_cov_mixture_5d(800, 14), 32),
        "nextafter1d": (np.concatenate([np.ones(20), np.full(20, np.nextafter(1.0, 2.0))]).reshape(-1, 1), 4),
        "dups2d": (np.tile([[0.25, -1.5]], (64, 1)), 4),
        "quantized3d": (np.round(g.random((900, 3)) * 6) / 6, 8),
        "uniform1d": (g.random((500, 1)), 7),
    }
    return out


def main():
    ref = load_reference()
    if ref is None:
        sys.exit("oracle/_ref/libdfgt_ref.so is not available")
    # trees
    trees = {}
    for name, (x, leaf) in datasets().items():
        t = ref.tree(x, leaf)
        trees[f"{name}__x"] = x
        trees[f"{name}__leaf"] = np.array(leaf)
        for f in t.fields():
            trees[f"{name}__{f}"] = getattr(t, f)
    np.savez_compressed(os.path.join(HERE, "trees.npz"), **trees)

    # sums (Q = R unless noted), reference DFGT with leaf 32 and explicit h
    sums, cv = {}, {}
    cases = [("cfg1", datagen.config(1, 0.12)), ("cfg2", datagen.config(2, 0.03)),
             ("cfg3", datagen.config(3, 0.008)), ("cfg4", datagen.config(4, 0.012))]
    for name, w in cases:
        x = w.refs
        sums[f"{name}__x"] = x
        scales = w.scales if len(w.scales) > 1 else (0.5, 1.0, 2.0)
        sums[f"{name}__h"] = np.array([s * w.h_s for s in scales])
        for eps in w.epsilons:
            eng = ref.engine(x, eps=eps, leaf=32)
            for i, s in enumerate(scales):
                h = s * w.h_s
                for tag, hh in (("h", h), ("2h", 2 * h)):
                    out, st = eng.compute(hh)
                    key = f"{name}__eps{eps}__{i}__{tag}"
                    sums[key + "__dfgt"] = out
                    sums[key + "__stats"] = st
                    if eps == w.epsilons[0]:
                        sums[f"{name}__{i}__{tag}__naive"] = ref.naive_kde(x, x, hh)
                d = f"{name}__eps{eps}__{i}"
                lk, cl = ref.lkcv(x, h, sums[d + "__h__dfgt"])
                ls = ref.lscv(x, h, sums[d + "__h__dfgt"], 2 * h, sums[d + "__2h__dfgt"])
                nlk, ncl = ref.lkcv(x, h, sums[f"{name}__{i}__h__naive"])
                nls = ref.lscv(x, h, sums[f"{name}__{i}__h__naive"], 2 * h,
                               sums[f"{name}__{i}__2h__naive"])
                cv[d] = {"h": h, "lk": lk, "lk_clamped": cl, "ls": ls, "naive_lk": nlk,
                         "naive_lk_clamped": ncl, "naive_ls": nls}
            eng.close()
    # Q != R (test_engine.cpp:87-99 analogue)
    g = np.random.default_rng(31)
    r = datagen.clustered_3d(700, 31)
    q = g.random((350, 3))
    sums["qr__r"], sums["qr__q"] = r, q
    for i, h in enumerate((0.05, 0.2, 2.0)):
        out, st = ref.dfgt(r, h, q=q, eps=0.001, leaf=20)
        sums[f"qr__{i}__dfgt"], sums[f"qr__{i}__stats"] = out, st
        sums[f"qr__{i}__naive"] = ref.naive_kde(q, r, h)
    sums["qr__h"] = np.array([0.05, 0.2, 2.0])
    np.savez_compressed(os.path.join(HERE, "sums.npz"), **sums)
    with open(os.path.join(HERE, "cv.json"), "w") as f:
        json.dump(cv, f, indent=1, sort_keys=True)

    # series primitives
    ser = {}
    rng = np.random.default_rng(5)
    for d, p in ((1, 8), (2, 6), (3, 4), (5, 2), (2, 3)):
        S = ref.series(d, p)
        T = p ** d
        pos, par, pdim, deg, invf = S.terms()
        k = f"d{d}p{p}"
        ser[k + "__terms"] = np.stack([pos, par, pdim, deg])
        ser[k + "__invf"] = invf
        c = rng.random(d)
        pts = c + 0.2 * (rng.random((13, d)) - 0.5)
        h = 0.3
        M = S.moments(pts, c, h)
        ser[k + "__pts"], ser[k + "__c"], ser[k + "__M"] = pts, c, M
        c2 = c + 0.1 * rng.random(d)
        ser[k + "__c2"] = c2
        ser[k + "__f2f"] = S.f2f(M, c, c2, h)
        q = c + 0.9 * rng.random(d)
        L0 = rng.random(T)
        ser[k + "__q"], ser[k + "__L0"] = q, L0
        ev_ff, ev_loc, dl, f2l, l2l = [], [], [], [], []
        for order in range(1, p + 1):
            ev_ff.append(S.eval_farfield(M, c, q, h, order))
            dl.append(S.direct_local(pts, q, h, order, L0))
            f2l.append(S.f2l(M, c, q, h, order, L0))
            l2l.append(S.l2l(L0, q, c2, h, order))
            ev_loc.append(S.eval_local(L0, c2, q, h, order))
        ser[k + "__eval_ff"] = np.array(ev_ff)
        ser[k + "__direct_local"] = np.array(dl)
        ser[k + "__f2l"] = np.array(f2l)
        ser[k + "__l2l"] = np.array(l2l)
        ser[k + "__eval_local"] = np.array(ev_loc)
    np.savez_compressed(os.path.join(HERE, "series.npz"), **ser)

    # truncation
    tr = []
    rng = np.random.default_rng(9)
    for _ in range(300):
        d = int(rng.integers(1, 6))
        p_max = [8, 6, 4, 2, 2][d - 1]
        nq, nr = float(rng.integers(1, 5000)), float(rng.integers(1, 5000))
        sq, sr = rng.uniform(0, 0.3), rng.uniform(0, 0.3)
        h = 10 ** rng.uniform(-2, 0)
        tau = 10 ** rng.uniform(-3, 2) * nr
        cm = int(rng.integers(0, 2))
        kind, order = ref.choose_best_method(nq, nr, sq, sr, h, tau, p_max, d, cm)
        r_ = rng.uniform(0.01, 0.95)
        pp = int(rng.integers(1, 9))
        tr.append({"args": [nq, nr, sq, sr, h, tau, p_max, d, cm], "kind": kind, "order": order,
                   "ff": [nr, r_, pp, d, ref.farfield_error_bound(nr, r_, pp, d)],
                   "f2l": [nr, r_ / 2, pp, d, ref.f2l_error_bound(nr, r_ / 2, pp, d)]})
    with open(os.path.join(HERE, "truncation.json"), "w") as f:
        json.dump(tr, f)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
