import sys; sys.path.insert(0,'.')
import paper_1102_2878_b200 as dfgtb
from paper_1102_2878_b200 import datagen
w=datagen.config(2)
e=dfgtb.DualTreeEngine(w.refs, config=dfgtb.EngineConfig(leaf_threshold=32))
for i in range(3):
    rows=e.sweep(w.scales, w.h_s)
    print(e.last_timings(), sum(r.seconds for r in rows)/len(rows))
