#!/usr/bin/env python
"""Full-size reference CV fixtures (BASELINE configs 1-4 at their stated N).

Runs the UNMODIFIED reference compiled from /root/reference (oracle/_ref/
libdfgt_ref.so) -- one single-threaded DualTreeEngine::compute per (config, eps,
bandwidth), spread over the host cores as processes -- on the exact bytes
paper_1102_2878_b200.datagen produces, and stores per row:

  lk, lk_clamped, ls      lkcv_from_sums / lscv_from_sums on the reference's sums
                          (cv.cpp:61-97; conv kernel 2h, cv.cpp:27-30)
  sum_h, sum_2h           sum over queries of the reference's G_h / G_2h
                          (a size-independent checksum: |sum_gpu - sum_ref| <= 2 eps sum_exact)
  seconds_h, seconds_2h   single-core reference compute time

plus the SHA-256 of the input points, so the GPU box (where /root/reference does not
exist) can check that its datagen reproduced the same bytes.  Output:
tests/golden/fullsize_cv.json.  tests/test_gpu_fullsize.py consumes it.

  python tests/golden/make_fullsize.py [--configs 1,2,3,4] [--procs 8]
"""
import argparse
import hashlib
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from paper_1102_2878_b200 import datagen  # noqa: E402


def sha(x: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(x, dtype=np.float64).tobytes()).hexdigest()


def _task(args):
    k, eps, h = args
    from oracle import load_reference
    ref = load_reference()
    w = datagen.config(k)
    t0 = time.perf_counter()
    eng = ref.engine(w.refs, eps=eps, leaf=w.leaf, p_max=w.p_max)
    sums, st = eng.compute(h)
    eng.close()
    return sums, time.perf_counter() - t0, st


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--configs", default="1,2,3,4")
    p.add_argument("--procs", type=int, default=os.cpu_count())
    p.add_argument("--out", default=os.path.join(HERE, "fullsize_cv.json"))
    a = p.parse_args()
    from oracle import load_reference
    ref = load_reference()
    if ref is None:
        sys.exit("oracle/_ref/libdfgt_ref.so is not available")
    out = json.load(open(a.out)) if os.path.exists(a.out) else {}
    for k in [int(c) for c in a.configs.split(",")]:
        w = datagen.config(k)
        x = w.refs
        hs = [s * w.h_s for s in w.scales]
        jobs = [(k, eps, hh) for eps in w.epsilons for h in hs for hh in (h, 2 * h)]
        t0 = time.perf_counter()
        with ProcessPoolExecutor(a.procs) as ex:
            res = list(ex.map(_task, jobs))
        wall = time.perf_counter() - t0
        by = {(j[1], j[2]): r for j, r in zip(jobs, res)}
        ent = {"name": w.name, "N": int(x.shape[0]), "D": int(x.shape[1]), "sha256": sha(x),
               "h_s": w.h_s, "scales": list(w.scales), "leaf": w.leaf,
               "p_max": ref.default_p_max(x.shape[1]) if not w.p_max else w.p_max,
               "wall_s": wall, "procs": a.procs, "rows": {}}
        for eps in w.epsilons:
            rows = []
            for s, h in zip(w.scales, hs):
                g1, t1, st1 = by[(eps, h)]
                g2, t2, st2 = by[(eps, 2 * h)]
                lk, cl = ref.lkcv(x, h, g1)
                ls = ref.lscv(x, h, g1, 2 * h, g2)
                rows.append({"scale": s, "h": h, "lk": lk, "lk_clamped": int(cl), "ls": ls,
                             "sum_h": float(np.sum(g1)), "sum_2h": float(np.sum(g2)),
                             "seconds_h": t1, "seconds_2h": t2,
                             "kernel_evaluations_h": int(st1[0]),
                             "kernel_evaluations_2h": int(st2[0])})
            ent["rows"][str(eps)] = rows
            lks = [r["lk"] for r in rows]
            lss = [r["ls"] for r in rows]
            ent.setdefault("h_star", {})[str(eps)] = {
                "lk": rows[int(np.argmax(lks))]["h"], "ls": rows[int(np.argmin(lss))]["h"]}
        out[f"cfg{k}"] = ent
        print(f"cfg{k}: {len(jobs)} reference computes in {wall:.1f} s on {a.procs} processes",
              flush=True)
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
