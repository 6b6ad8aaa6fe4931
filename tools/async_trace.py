import sys, os
sys.path.insert(0, '.')
import paper_1102_2878_b200 as dfgtb
from paper_1102_2878_b200 import datagen
w = datagen.config(int(sys.argv[1]))
e = dfgtb.DualTreeEngine(w.refs, config=dfgtb.EngineConfig(leaf_threshold=32))
e.sweep(w.scales, w.h_s)
print("--- second", file=sys.stderr, flush=True)
e.sweep(w.scales, w.h_s)
