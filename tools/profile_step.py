#!/usr/bin/env python
"""One warm-up pass + one measured pass of a config's workload, for ncu launch lists.
Q = R configs run the on-device CV sweep (dfgtb_sweep); config 5 (Q != R) runs its
three bandwidths through one compute_batch.  Prints the library launch counter
before and after the measured pass so the launch list can be cut to exactly it.

  python tools/profile_step.py [--config 2]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", type=int, default=2)
    a = p.parse_args()
    import paper_1102_2878_b200 as dfgtb
    from paper_1102_2878_b200 import _capi, datagen
    w = datagen.config(a.config)
    e = dfgtb.DualTreeEngine(w.refs, config=dfgtb.EngineConfig(epsilon=w.epsilons[0], leaf_threshold=32))
    if w.queries is None:
        run = lambda: e.sweep(w.scales, w.h_s)  # noqa: E731
    else:
        hs = [s * w.h_s for s in w.scales]
        run = lambda: e.compute_batch(w.queries, hs)  # noqa: E731
    run()  # warm-up
    l0 = _capi.lib.dfgtb_launch_count(e.handle)
    t0 = time.perf_counter()
    run()
    t1 = time.perf_counter()
    l1 = _capi.lib.dfgtb_launch_count(e.handle)
    print(f"launches_before={l0} launches_after={l1} wall_s={t1 - t0:.6f}")


if __name__ == "__main__":
    main()
