#!/usr/bin/env python
"""Wall-clock breakdown of the end-to-end public-API path on config 2:
engine creation (H2D + GPU tree + moments), sweep (first / second), destroy."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_1102_2878_b200 as dfgtb
    from paper_1102_2878_b200 import datagen
    w = datagen.config(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
    cfg = dfgtb.EngineConfig(epsilon=0.01, leaf_threshold=32)
    for it in range(5):
        t0 = time.perf_counter()
        e = dfgtb.DualTreeEngine(w.refs, dfgtb.Mode.series, cfg)
        t1 = time.perf_counter()
        e.sweep(w.scales, w.h_s)
        t2 = time.perf_counter()
        e.sweep(w.scales, w.h_s)
        t3 = time.perf_counter()
        tree_ms = e.last_timings()["tree_ms"]
        e.close()
        t4 = time.perf_counter()
        print(f"iter {it}: create {1e3*(t1-t0):.2f} ms (tree+moments device {tree_ms:.2f}), "
              f"sweep1 {1e3*(t2-t1):.2f} ms, sweep2 {1e3*(t3-t2):.2f} ms, destroy {1e3*(t4-t3):.2f} ms",
              flush=True)


if __name__ == "__main__":
    main()
