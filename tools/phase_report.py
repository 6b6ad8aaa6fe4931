#!/usr/bin/env python
"""Per-bandwidth phase timings and traversal statistics of the GPU engine.

  python tools/phase_report.py [--config 2] [--scale 1.0] [--check]

Prints one JSON line per compute (h and 2h at every sweep scale): device ms per
phase (events on the engine stream), TraversalStats, and with --check the max
relative error against the GPU exhaustive FP64 sum on a seeded query subsample.
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", type=int, default=2)
    p.add_argument("--scale", type=float, default=1.0)
    p.add_argument("--check", action="store_true")
    p.add_argument("--sub", type=int, default=4096)
    a = p.parse_args()
    import paper_1102_2878_b200 as dfgtb
    from paper_1102_2878_b200 import datagen
    w = datagen.config(a.config, a.scale)
    import time
    for i in range(3):  # engine construction cost (upload + GPU tree + moments)
        t0 = time.perf_counter()
        e = dfgtb.DualTreeEngine(w.refs, config=dfgtb.EngineConfig(leaf_threshold=32))
        t1 = time.perf_counter()
        tree_ms = e.last_timings()["tree_ms"]
        e.close()
        t2 = time.perf_counter()
        print(json.dumps({"create_s": t1 - t0, "tree_ms": tree_ms, "destroy_s": t2 - t1}))
    for eps in w.epsilons:
        e = dfgtb.DualTreeEngine(w.refs, config=dfgtb.EngineConfig(epsilon=eps, leaf_threshold=32))
        print(json.dumps({"config": w.name, "n": int(w.refs.shape[0]), "h_s": w.h_s, "eps": eps,
                          "tree_ms": e.last_timings()["tree_ms"]}))
        q = w.queries
        rng = np.random.default_rng(7)
        for s in w.scales:
            for mult in ((1.0, 2.0) if q is None else (1.0,)):
                h = s * w.h_s * mult
                e.compute(q, h)  # warm
                out = e.compute(q, h)
                rec = {"scale": s, "h": h, **e.last_timings(), **vars(e.last_stats())}
                if a.check:
                    qs = w.refs if q is None else q
                    idx = rng.choice(qs.shape[0], min(a.sub, qs.shape[0]), replace=False)
                    ex = dfgtb.naive_kde(qs[idx], w.refs, h)
                    ok = ex > 0
                    rec["max_rel_err"] = float(np.max(np.abs(out[idx][ok] - ex[ok]) / ex[ok]))
                    rec["exact_zero"] = int((~ok).sum())
                print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
