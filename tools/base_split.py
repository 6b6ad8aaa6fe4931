#!/usr/bin/env python
"""Per-bandwidth split of the base case between the FP32 and the FP64 kernels
(tasks and (q, r) pairs), one compute per bandwidth of a config's sweep.

  python tools/base_split.py [--config 2]
"""
import argparse
import ctypes
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
    e = dfgtb.DualTreeEngine(w.refs, config=dfgtb.EngineConfig(epsilon=w.epsilons[0], leaf_threshold=32))
    ta, tb, pa, pb = ctypes.c_int(), ctypes.c_int(), ctypes.c_uint64(), ctypes.c_uint64()
    tot = [0, 0]
    for s in w.scales:
        for f in ((1.0, 2.0) if w.queries is None else (1.0,)):
            h = s * f * w.h_s
            e.compute(w.queries, h)
            _capi.check(_capi.lib.dfgtb_last_base_split(e.handle, ctypes.byref(ta), ctypes.byref(tb),
                                                        ctypes.byref(pa), ctypes.byref(pb)))
            tot[0] += pa.value
            tot[1] += pb.value
            print(f"h={h:.4g} f32 tasks {ta.value} pairs {pa.value:.4g} | fp64 tasks {tb.value} pairs {pb.value:.4g}")
    print(f"total pairs f32 {tot[0]:.4g} fp64 {tot[1]:.4g} (f32 share {tot[0] / max(1, sum(tot)):.3f})")


if __name__ == "__main__":
    main()
