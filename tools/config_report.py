#!/usr/bin/env python
"""Full-size run of every BASELINE.json config on one GPU, with the north star's
correctness check (a) on ALL queries and per-bandwidth throughput.

For each config (datagen.config(k), full N) and each epsilon:
  * one engine (tree + moments built on the GPU, timed),
  * all of the config's bandwidths (h, and 2h where CV_LS needs it) through one
    lock-step batch, timed on the host around the call (includes the D2H of sums),
  * exact FP64 sums for EVERY query from the GPU exhaustive kernel (k_naive), itself
    pinned against the oracle's C naive sum on a 128-query subsample,
  * max relative error over queries (exact-zero queries counted separately),
  * for Q = R configs: the on-device CV sweep (dfgtb_sweep) timed with CUDA events
    and its scores.

  python tools/config_report.py [--configs 1,2,3,4,5] [--out gpurun_out/configs.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--configs", default="1,2,3,4,5")
    p.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "configs.json"))
    p.add_argument("--pin", type=int, default=128, help="queries checked against the C oracle")
    a = p.parse_args()
    import paper_1102_2878_b200 as dfgtb
    from paper_1102_2878_b200 import datagen
    from oracle import load_oracle
    orc = load_oracle()
    report = []
    for k in [int(x) for x in a.configs.split(",")]:
        w = datagen.config(k)
        q = w.queries
        nq = (q if q is not None else w.refs).shape[0]
        hs = [s * w.h_s for s in w.scales]
        batch = hs + ([2 * h for h in hs] if "ls" in w.scores else [])
        rng = np.random.default_rng(7)
        pin_idx = np.sort(rng.choice(nq, size=min(a.pin, nq), replace=False))
        qq = q if q is not None else w.refs
        # exact sums, once per bandwidth (GPU FP64 exhaustive kernel), pinned to the oracle
        t0 = time.perf_counter()
        exact = np.stack([dfgtb.naive_kde(qq, w.refs, h) for h in batch])
        t_naive = time.perf_counter() - t0
        pin_err = 0.0
        for b, h in enumerate(batch[: min(3, len(batch))]):
            o = orc.naive_kde(qq[pin_idx], w.refs, h)
            e = exact[b, pin_idx]
            nz = o > 0
            if nz.any():
                pin_err = max(pin_err, float(np.max(np.abs(e[nz] - o[nz]) / o[nz])))
        for eps in w.epsilons:
            cfg = dfgtb.EngineConfig(epsilon=eps, leaf_threshold=w.leaf, p_max=w.p_max or None)
            # config 5 declares fp32 inputs: feed float32 arrays (widened exactly on device)
            r_in = w.refs.astype(np.float32) if k == 5 else w.refs
            q = w.queries.astype(np.float32) if (k == 5 and w.queries is not None) else w.queries
            t0 = time.perf_counter()
            eng = dfgtb.DualTreeEngine(r_in, dfgtb.Mode.series, cfg)
            t_build = time.perf_counter() - t0
            eng.compute_batch(q, batch)  # warm-up
            t0 = time.perf_counter()
            sums = eng.compute_batch(q, batch)
            t_batch = time.perf_counter() - t0
            stats = eng.batch_stats()
            rows = []
            for b, h in enumerate(batch):
                ex, got = exact[b], sums[b]
                zero = ex <= 0
                rel = np.abs(got[~zero] - ex[~zero]) / ex[~zero]
                rows.append({
                    "h": h, "scale_of_hs": h / w.h_s,
                    "max_rel_err": float(rel.max()) if rel.size else 0.0,
                    "n_over_eps": int(np.sum(rel > eps)),
                    "exact_zero": int(zero.sum()), "zero_ok": bool(np.all(got[zero] == 0.0)),
                    "kernel_evaluations": stats[b].kernel_evaluations if b < len(stats) else None,
                })
            sweep = None
            if q is None and w.scales:
                import torch
                from paper_1102_2878_b200 import _capi
                stream = torch.cuda.ExternalStream(_capi.lib.dfgtb_stream(eng.handle))
                eng.sweep(w.scales, w.h_s)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                srows = eng.sweep(w.scales, w.h_s)
                e1.record(stream)
                e1.synchronize()
                sweep = {"ms": e0.elapsed_time(e1), "bandwidths": 2 * len(w.scales),
                         "queries_per_s": 2 * len(w.scales) * nq / (e0.elapsed_time(e1) * 1e-3),
                         "rows": [{"h": r.h, "lk": r.lk_score, "lk_clamped": r.lk_clamped,
                                   "ls": r.ls_score, "base_ms": r.base_ms,
                                   "base_pairs": r.base_pairs} for r in srows]}
                lk = [r.lk_score for r in srows]
                ls = [r.ls_score for r in srows]
                sweep["h_star_lk"] = srows[int(np.argmax(lk))].h
                sweep["h_star_ls"] = srows[int(np.argmin(ls))].h
            eng.close()
            ent = {"config": k, "name": w.name, "N_refs": int(w.refs.shape[0]), "N_queries": int(nq),
                   "D": int(w.refs.shape[1]), "eps": eps, "bandwidths": len(batch),
                   "engine_build_s": t_build, "batch_s": t_batch,
                   "batch_queries_per_s": len(batch) * nq / t_batch,
                   "max_rel_err": max(r["max_rel_err"] for r in rows),
                   "n_over_eps": sum(r["n_over_eps"] for r in rows),
                   "exact_zero": sum(r["exact_zero"] for r in rows),
                   "naive_vs_oracle_max_rel": pin_err, "naive_s": t_naive,
                   "rows": rows, "sweep": sweep}
            report.append(ent)
            print(json.dumps({x: ent[x] for x in ent if x not in ("rows", "sweep")}), flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(report, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
