"""Step time and accuracy vs DFGTB_TRAV_START_DEPTH (run once per depth: the env is read once)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1102_2878_b200 as dfgtb
from paper_1102_2878_b200 import _capi, datagen
k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = datagen.config(k)
e = dfgtb.DualTreeEngine(w.refs, config=dfgtb.EngineConfig(leaf_threshold=32))
st = torch.cuda.ExternalStream(_capi.lib.dfgtb_stream(e.handle))
for _ in range(3): e.sweep(w.scales, w.h_s)
ms = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st); e.sweep(w.scales, w.h_s); b.record(st); b.synchronize(); ms.append(a.elapsed_time(b))
t = e.last_timings()
hs = [s * w.h_s for s in w.scales] + [2 * s * w.h_s for s in w.scales]
g = e.compute_batch(None, hs)
ex = np.stack([dfgtb.naive_kde(w.refs, w.refs, h) for h in hs])
print(json.dumps({"depth": os.environ.get("DFGTB_TRAV_START_DEPTH", "0"), "ms": float(np.mean(ms)), "trav": t["traverse_ms"],
                  "base": t["base_ms"], "local": t["local_ms"], "ff": t["farfield_ms"], "final": t["final_ms"],
                  "maxrel": float(np.max(np.abs(g - ex) / ex))}))
