#!/usr/bin/env python
"""SHA-256 of a config's kernel sums (every bandwidth of its sweep, h and 2h for Q = R)
and the summed traversal statistics: two library builds whose traversal decisions are
identical print identical lines.

  DFGTB_LIB=path/to/libdfgtb.so python tools/sums_hash.py [config]
"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_1102_2878_b200 as dfgtb  # noqa: E402
from paper_1102_2878_b200 import datagen  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = datagen.config(k)
e = dfgtb.DualTreeEngine(w.refs, config=dfgtb.EngineConfig(epsilon=w.epsilons[0], leaf_threshold=32))
hs = [s * f * w.h_s for s in w.scales for f in ((1.0, 2.0) if w.queries is None else (1.0,))]
sums = e.compute_batch(w.queries, hs)
print("cfg", k, "sha256", hashlib.sha256(np.ascontiguousarray(sums).tobytes()).hexdigest()[:16], e.last_stats())
