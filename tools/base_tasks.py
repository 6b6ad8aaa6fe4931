import sys, os, ctypes as C
sys.path.insert(0, '.')
import paper_1102_2878_b200 as dfgtb
from paper_1102_2878_b200 import _capi, datagen
w = datagen.config(2)
e = dfgtb.DualTreeEngine(w.refs, config=dfgtb.EngineConfig(leaf_threshold=32))
e.sweep(w.scales, w.h_s)
ta, tb, pa, pb = C.c_int(), C.c_int(), C.c_uint64(), C.c_uint64()
_capi.check(_capi.lib.dfgtb_last_base_split(e.handle, C.byref(ta), C.byref(tb), C.byref(pa), C.byref(pb)))
print("f32 tasks", ta.value, "pairs", pa.value, "per task", pa.value / max(1, ta.value), "| fp64 tasks", tb.value, "pairs", pb.value, pb.value / max(1, tb.value))
