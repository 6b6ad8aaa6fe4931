#!/usr/bin/env python
"""Wall / event time of config 5's public-API call (1M x 1M, 3 bandwidths, float32 pinned
queries in, float64 pinned sums out: H2D, query tree, batch, D2H), per step.

  [DFGTB_LIB=...] python tools/cfg5_api.py [steps]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_1102_2878_b200 as dfgtb
    from paper_1102_2878_b200 import datagen
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    w = datagen.config(5)
    eng = dfgtb.DualTreeEngine(w.refs.astype(np.float32), dfgtb.Mode.series,
                               dfgtb.EngineConfig(epsilon=0.01, leaf_threshold=32))
    hs = [s * w.h_s for s in w.scales]
    q = torch.empty(w.queries.shape, dtype=torch.float32, pin_memory=True).numpy()
    q[:] = w.queries
    o = torch.empty((len(hs), w.queries.shape[0]), dtype=torch.float64, pin_memory=True).numpy()
    eng.compute_batch(q, hs, out=o)
    for _ in range(steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.compute_batch(q, hs, out=o)
        t1 = time.perf_counter()
        print(f"call {1e3 * (t1 - t0):.2f} ms, device batch {eng.last_timings()['total_ms']:.2f} ms", flush=True)


if __name__ == "__main__":
    main()
