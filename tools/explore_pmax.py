"""Which (N, cost model, eps, h) make the 5-D traversal choose series methods (p_max 8)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1102_2878_b200 as dfgtb
from paper_1102_2878_b200 import datagen
for d, p in ((5, 8), (5, 3), (3, 1), (5, 1)):
    for n in (1500, 20000):
        x = datagen.full_cov_mixture_5d(n, 77) if d == 5 else datagen.clustered_3d(n, 77)
        hs = datagen.silverman_h(x) * np.array([0.3, 1, 3, 10, 30])
        for cm in (0, 1):
            for eps in (1e-2, 1e-3, 1e-4):
                t = time.time()
                with dfgtb.DualTreeEngine(x, config=dfgtb.EngineConfig(epsilon=eps, leaf_threshold=32, p_max=p, cost_model=cm)) as e:
                    e.compute_batch(None, hs)
                    st = e.batch_stats()
                print(d, p, n, cm, eps, [(s.prunes_farfield, s.prunes_direct_local, s.prunes_far_to_local, s.prunes_finite_diff) for s in st], round(time.time() - t, 2), flush=True)
