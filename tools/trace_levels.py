#!/usr/bin/env python
"""Per-level timing of the persistent traversal kernel (DFGTB_TRACE=1): runs one
batched config-2 sweep and prints the %globaltimer phase stamps of k_traverse."""
import os
import sys

os.environ["DFGTB_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1102_2878_b200 as dfgtb  # noqa: E402
from paper_1102_2878_b200 import datagen  # noqa: E402

w = datagen.config(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
e = dfgtb.DualTreeEngine(w.refs, config=dfgtb.EngineConfig(leaf_threshold=32))
e.sweep(w.scales, w.h_s)
print("---- second sweep ----", file=sys.stderr, flush=True)
e.sweep(w.scales, w.h_s)
