import sys; sys.path.insert(0,'.')
import numpy as np
import paper_1102_2878_b200 as dfgtb
from paper_1102_2878_b200 import datagen
for n, seed in ((20000, 605), (20000, 77), (40000, 605)):
    x = datagen.full_cov_mixture_5d(n, seed)
    hs = datagen.silverman_h(x) * np.array([1, 3, 10, 30, 100])
    for p in (2, 5, 8):
        for eps in (1e-2, 1e-3):
            with dfgtb.DualTreeEngine(x, config=dfgtb.EngineConfig(epsilon=eps, leaf_threshold=32, p_max=p, cost_model=1)) as e:
                e.compute_batch(None, hs); st = e.batch_stats()
            print(n, seed, p, eps, [(s.prunes_farfield, s.prunes_direct_local, s.prunes_finite_diff) for s in st], flush=True)
for p in (3, 5):
    x = datagen.full_cov_mixture_5d(1500, 900 + 5 + p)
    for sc in (10, 30, 100):
        h = datagen.silverman_h(x) * sc
        e = dfgtb.DualTreeEngine(x, config=dfgtb.EngineConfig(epsilon=0.01, leaf_threshold=32, p_max=p, cost_model=1)); e.compute(None, h); s = e.last_stats()
        print(1500, p, sc, s.prunes_farfield, s.prunes_direct_local, s.prunes_finite_diff)
