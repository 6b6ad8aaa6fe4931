#!/usr/bin/env python
"""One warm-up sweep + one measured sweep of the bench workload (config 2), for
ncu launch lists.  Prints the library launch counter before and after the
measured sweep so the launch list can be cut to exactly that step.

  python tools/profile_step.py [--config 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", type=int, default=2)
    a = p.parse_args()
    import paper_1102_2878_b200 as dfgtb
    from paper_1102_2878_b200 import _capi, datagen
    w = datagen.config(a.config)
    e = dfgtb.DualTreeEngine(w.refs, config=dfgtb.EngineConfig(epsilon=0.01, leaf_threshold=32))
    e.sweep(w.scales, w.h_s)  # warm-up
    l0 = _capi.lib.dfgtb_launch_count(e.handle)
    rows = e.sweep(w.scales, w.h_s)
    l1 = _capi.lib.dfgtb_launch_count(e.handle)
    print(f"launches_before={l0} launches_after={l1} sweep_device_s={sum(r.seconds for r in rows):.6f}")


if __name__ == "__main__":
    main()
