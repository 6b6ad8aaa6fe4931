#!/usr/bin/env python
"""Benchmark: DFGT kernel-sum queries/sec on BASELINE config 2 (one B200).

Workload (BASELINE.json configs[1]): Q = R = 50,000 points, D = 2,
16-component clipped Gaussian mixture (seeded synthetic), eps = 0.01, leaf 32,
p_max = 6.  One STEP = the full CV bandwidth sweep: 9 bandwidths h = h_s 10^k,
k in {-3,-2,-1,-0.5,0,0.5,1,2,3}, each with kernel sums at h and at 2h (18 sums of
50k queries) and CV_LK + CV_LS reduced on the device.  Metric = queries/sec per h
= 18 * 50,000 / step time (whole job over all ranks).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--quick]

--impl reference times the reference's own CPU implementation (compiled from
/root/reference into oracle/_ref) on the host cores, same workload.  N > 1 (torchrun)
runs ONE sweep with its queries sharded over the ranks (strong scaling, one NCCL
all_reduce of 3 CV partials per bandwidth).  Besides the headline, the N = 1 line
carries: per-h timings, the FP64-only (DFGTB_NO_F32) number, device-timed cfg3 and
cfg5 records, tree/moment HBM fractions, and a parity block (max relative error over
every query, CV vs the reference's scores from the cpu_baseline leg, h*, tree bit-exact).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gaussian KDE kernel-sum queries/sec (Q=R, eps=1e-2) per h; % of exp/FP64 roofline"
UNIT = "queries/s"
FP64_INSTR_PER_PAIR = {1: 21, 2: 23, 3: 25, 4: 27, 5: 29}  # 2D+19, see DESIGN.md


def workload(rank: int = 0):
    from paper_1102_2878_b200 import datagen
    return datagen.config(2)


# --------------------------------------------------------------------- reference
def _ref_one(args):
    refs, h, eps, leaf = args
    from oracle import load_reference
    ref = load_reference()
    t0 = time.perf_counter()
    eng = ref.engine(refs, eps=eps, leaf=leaf)
    sums, _ = eng.compute(h)
    eng.close()
    return sums, time.perf_counter() - t0


def reference_sweep(w, cores: int):
    """The reference's bandwidth sweep for both CV scores: one reference engine per
    (h | 2h) compute, `cores` processes (the engine is single-threaded, engine.hpp:85)."""
    import multiprocessing as mp
    hs = [s * w.h_s for s in w.scales]
    jobs = [(w.refs, h, 0.01, 32) for h in hs] + [(w.refs, 2 * h, 0.01, 32) for h in hs]
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(min(cores, len(jobs))) as pool:
        res = pool.map(_ref_one, jobs, chunksize=1)
    wall = time.perf_counter() - t0
    from oracle import load_reference
    ref = load_reference()  # the reference's own lkcv_from_sums / lscv_from_sums (cv.cpp:61-97)
    n = len(hs)
    scores = []
    for i, h in enumerate(hs):
        lk, cl = ref.lkcv(w.refs, h, res[i][0])
        ls = ref.lscv(w.refs, h, res[i][0], 2 * h, res[n + i][0])
        scores.append((h, lk, cl, ls))
    return wall, scores, sum(r[1] for r in res)


def run_reference(a, rank, world):
    if rank != 0:
        return
    from oracle import load_reference
    if load_reference() is None:
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libdfgt_ref.so not built (needs /root/reference at build time)"}))
        return
    w = workload(0)
    cores = os.cpu_count() or 1
    n_q = 2 * len(w.scales) * w.refs.shape[0]
    for _ in range(a.warmup):
        reference_sweep(w, cores)
    times = []
    for _ in range(a.steps):
        wall, _, _ = reference_sweep(w, cores)
        times.append(wall)
    t = float(np.mean(times))
    v = n_q / t
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(w, world),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": min(cores, 18), "kind": "reference",
                         "cpu": cpu_model(),
                         "sample": "full cfg2 sweep per step: 18 reference DualTreeEngine computes "
                                   "(9 scales x {h, 2h}), one engine per compute, "
                                   f"{min(cores, 18)} processes on the host cores"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def config_block(w, world):
    return {"workload": f"{w.name}: CV sweep 9 x (h, 2h) kernel sums + CV_LK/CV_LS",
            "N": int(w.refs.shape[0]), "D": int(w.refs.shape[1]), "eps": 0.01, "leaf": 32,
            "p_max": 6, "bandwidths": 18, "global_batch": int(18 * w.refs.shape[0]),
            "l2": "flushed between timed steps (256 MiB device write)",
            "parallelism": f"query-sharded x{world}" if world > 1 else "single"}


# -------------------------------------------------------------------------- ours
class Clocks:
    """SM clock and clock-event reasons sampled DURING the timed region: an NVML
    polling thread (~1 ms period; the timed region is only milliseconds long, too
    short for `nvidia-smi -lms`).  NVML calls release the GIL (ctypes)."""

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4), ("hw_power_brake_slowdown", 0x80))

    def __init__(self, idx):
        self.idx = idx
        self.rows = []
        self.err = None

    def _run(self):
        import pynvml
        try:
            while not self.stop:
                sm = pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.rows.append((sm, rs))
                time.sleep(0.001)
        except Exception as e:  # pragma: no cover - reported in the line
            self.err = repr(e)

    def __enter__(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            phys = int(vis.split(",")[self.idx]) if vis and vis.split(",")[0].isdigit() else self.idx
            self.h = pynvml.nvmlDeviceGetHandleByIndex(phys)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:
            self.err = repr(e)
            self.th = None
            return self
        self.stop = False
        self.th = threading.Thread(target=self._run, daemon=True)
        self.th.start()
        while not self.rows and self.err is None and self.th.is_alive():  # first sample before timing
            time.sleep(0.0005)
        self.rows.clear()
        return self

    def __exit__(self, *a):
        if self.th is not None:
            self.stop = True
            self.th.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "error": self.err}
        sm = sorted(r[0] for r in self.rows)
        reasons = sorted({n for _, m in self.rows for n, bit in self.REASONS if m & bit})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": int(self.max_mhz), "reasons": reasons,
                "samples": len(self.rows), "sm_mhz_min": sm[0], "sampler": "nvml, ~1 ms period"}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def _events_ms(stream, fn, reps=1):
    """Device time (CUDA events on the engine stream) of fn(), mean over reps."""
    import torch
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        e1.synchronize()
        out.append(e0.elapsed_time(e1))
    return float(np.mean(out))


def hbm_peak():
    mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(mp))["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return 6526.8, "fallback (SURVEY 8(d))"


def parity_block(dfgtb, eng, w, ref_scores, ref_tree):
    """North-star checks on the benched workload itself, outside the timed region:
    (a) max relative error of the engine's sums over ALL queries and all 18 bandwidths
    against exact FP64 sums (GPU exhaustive kernel K12, pinned to the C oracle in
    tests/test_gpu_fullsize.py); (b) CV scores vs the reference's (its CPU sweep in the
    cpu_baseline leg) against the rigorous 2-eps bounds, and h*; (c) the GPU tree vs the
    reference's KdTree::build, bit for bit."""
    x = w.refs
    n, d = x.shape
    eps = 0.01
    hs = [s * w.h_s for s in w.scales]
    batch = hs + [2 * h for h in hs]
    exact = np.stack([dfgtb.naive_kde(x, x, h) for h in batch])
    sums = eng.compute_batch(None, batch)
    rel = np.abs(sums - exact) / exact
    out = {"max_rel_err": float(rel.max()), "eps": eps, "queries_checked": int(n),
           "bandwidths_checked": len(batch), "n_over_eps": int(np.sum(rel > eps)),
           "exact": "GPU FP64 exhaustive sums (k_naive) of every query"}
    rows = eng.sweep(w.scales, w.h_s)
    ik, il = dfgtb.DualTreeEngine.best(rows)
    out["h_star"] = {"lk": rows[ik].h, "ls": rows[il].h}
    if ref_scores is not None:
        ns = len(hs)
        cv, ls_ref, ls_b = [], [], []
        for i, (row, (h, lk_r, cl_r, ls_r)) in enumerate(zip(rows, ref_scores)):
            g1, g2 = exact[i], exact[ns + i]
            nh = (n - 1) * (2 * np.pi * h * h) ** (d / 2)
            nc = (n - 1) * (2 * np.pi * 4 * h * h) ** (d / 2)
            lsb = 2 * eps / n * float(np.sum(g2 / nc + 2 * g1 / nh))
            kappa = float(np.max(2 * eps * g1 / np.maximum(g1 - 1.0, 1e-300)))
            lk_ok = kappa < 0.5 and cl_r == 0 and row.lk_clamped == 0
            lkb = float(-np.mean(np.log1p(-2 * eps * g1 / (g1 - 1.0)))) if lk_ok else None
            cv.append({"h": h, "ls_gpu": row.ls_score, "ls_ref": ls_r, "ls_delta": abs(row.ls_score - ls_r),
                       "ls_bound": lsb, "ls_ok": abs(row.ls_score - ls_r) <= lsb * (1 + 1e-9),
                       "lk_gpu": row.lk_score, "lk_ref": lk_r, "lk_delta": abs(row.lk_score - lk_r),
                       "lk_bound": lkb, "lk_ok": (abs(row.lk_score - lk_r) <= lkb * (1 + 1e-9)) if lk_ok else None,
                       "lk_clamped_gpu": row.lk_clamped, "lk_clamped_ref": cl_r})
            ls_ref.append(ls_r)
            ls_b.append(lsb / 2)
        out["cv_vs_reference"] = cv
        out["cv_all_within_bound"] = all(r["ls_ok"] and r["lk_ok"] is not False for r in cv)
        kr = int(np.argmin(ls_ref))
        out["h_star_reference"] = {"ls": ref_scores[kr][0],
                                   "lk": ref_scores[int(np.argmax([r[1] for r in ref_scores]))][0]}
        out["h_star_ls_equal"] = rows[il].h == ref_scores[kr][0]
    if ref_tree is not None:
        gt = eng.reference_tree()
        out["tree_bit_exact"] = all(np.array_equal(getattr(gt, f), getattr(ref_tree, f)) for f in ref_tree.fields())
    return out


def config_records(dfgtb, flush, steps):
    """Device-timed sweeps of the largest Q = R config (cfg3, 200k 3-D, 18 bandwidths)
    and of the 1M x 1M config (cfg5, 3 bandwidths, float32 inputs), with their
    base-case rooflines -- reported beside the cfg2 headline, not instead of it."""
    import torch
    from paper_1102_2878_b200 import _capi, datagen
    peak_ex2 = _capi.lib.dfgtb_ex2_peak()
    recs = []
    for k in (3, 5):
        w = datagen.config(k)
        cfg = dfgtb.EngineConfig(epsilon=0.01, leaf_threshold=32)
        r_in = w.refs.astype(np.float32) if k == 5 else w.refs
        q_in = w.queries.astype(np.float32) if k == 5 else None
        nq = (w.queries if w.queries is not None else w.refs).shape[0]
        t0 = time.perf_counter()
        eng = dfgtb.DualTreeEngine(r_in, dfgtb.Mode.series, cfg)
        build_s = time.perf_counter() - t0
        stream = torch.cuda.ExternalStream(_capi.lib.dfgtb_stream(eng.handle))
        hs = [s * w.h_s for s in w.scales]
        if k == 5:
            nbw = len(hs)
            # pinned host buffers for the queries and the sums (reused every call)
            q_pin = torch.empty(q_in.shape, dtype=torch.float32, pin_memory=True).numpy()
            q_pin[:] = q_in
            o_pin = torch.empty((nbw, nq), dtype=torch.float64, pin_memory=True).numpy()
            fn = lambda: eng.compute_batch(q_pin, hs, out=o_pin)  # noqa: E731  (public API: H2D, query tree, D2H)
        else:
            nbw = 2 * len(hs)
            fn = lambda: eng.sweep(w.scales, w.h_s)  # noqa: E731
        fn()
        fn()  # two warm-up calls: the first grows the batch buffers, the second the pinned pools
        ms, dev_ms, base_ms, pairs = [], [], [], []
        for _ in range(steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            ms.append(_events_ms(stream, fn))
            t = eng.last_timings()
            dev_ms.append(t["total_ms"])
            base_ms.append(t["base_ms"])
            ta, tb, pa, pb = C.c_int(), C.c_int(), C.c_uint64(), C.c_uint64()
            _capi.check(_capi.lib.dfgtb_last_base_split(eng.handle, C.byref(ta), C.byref(tb),
                                                        C.byref(pa), C.byref(pb)))
            pairs.append(pa.value + pb.value)
        t_ms = float(np.mean(ms))
        rate = float(np.mean(pairs)) / (float(np.mean(base_ms)) * 1e-3)
        recs.append({"config": k, "workload": w.name, "N_refs": int(w.refs.shape[0]), "N_queries": int(nq),
                     "D": int(w.refs.shape[1]), "bandwidths": nbw,
                     "timed": "public API call incl. H2D of float32 queries (pinned), query tree and D2H of "
                              "sums (pinned)"
                              if k == 5 else "dfgtb_sweep, engine resident, CV on device",
                     "ms_per_step": t_ms, "queries_per_s": nbw * nq / (t_ms * 1e-3),
                     "device_ms_traversal_to_sums": float(np.mean(dev_ms)),
                     "engine_build_s": build_s,
                     "base_case": {"pairs_per_step": int(np.mean(pairs)), "ms_per_step": float(np.mean(base_ms)),
                                   "achieved_g_ex2_s": rate / 1e9, "frac_of_ex2_peak": rate / peak_ex2}})
        eng.close()
    return recs


def run_ours(a, rank, world, local_rank):
    import torch
    torch.cuda.set_device(local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        return run_sharded(a, rank, world, local_rank)
    import paper_1102_2878_b200 as dfgtb
    from paper_1102_2878_b200 import _capi

    w = workload(rank)
    n = w.refs.shape[0]
    cfg = dfgtb.EngineConfig(epsilon=0.01, leaf_threshold=32)
    eng = dfgtb.DualTreeEngine(w.refs, dfgtb.Mode.series, cfg)
    stream = torch.cuda.ExternalStream(_capi.lib.dfgtb_stream(eng.handle))
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MiB > L2
    peak_instr = _capi.lib.dfgtb_dfma_peak()
    peak_ex2 = _capi.lib.dfgtb_ex2_peak()
    exp_mode = _capi.lib.dfgtb_base_exp_mode(eng.handle)
    mufu = exp_mode >= 1

    def step():
        return eng.sweep(w.scales, w.h_s)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    l0 = _capi.lib.dfgtb_launch_count(eng.handle)
    ms, base_ms, base_pairs, rows = [], 0.0, 0, None
    f32_ms, fp64_ms = 0.0, 0.0
    phases = {}
    with Clocks(local_rank) as clk:
        for _ in range(a.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            rows = step()
            e1.record(stream)
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
            base_ms += sum(r.base_ms for r in rows)
            base_pairs += sum(r.base_pairs for r in rows)
            tm = eng.last_timings()
            f32_ms += tm["base_f32_ms"]
            fp64_ms += tm["base_fp64_ms"]
            for kname in ("traverse_ms", "moments_ms", "local_ms", "base_ms", "farfield_ms", "final_ms", "total_ms"):
                phases[kname] = phases.get(kname, 0.0) + tm[kname] / a.steps
    launches = _capi.lib.dfgtb_launch_count(eng.handle) - l0
    # the base-case pairs on each kernel (every step runs the same sweep)
    ta, tb, pa, pb = C.c_int(), C.c_int(), C.c_uint64(), C.c_uint64()
    _capi.check(_capi.lib.dfgtb_last_base_split(eng.handle, C.byref(ta), C.byref(tb), C.byref(pa), C.byref(pb)))
    torch.cuda.synchronize()
    t_step = float(np.mean(ms))
    value = 18 * n / (t_step * 1e-3)

    # e2e: public API with host buffers (pinned), engine build + sweep + scores back
    pinned = torch.empty(w.refs.shape, dtype=torch.float64, pin_memory=True)
    pinned.numpy()[:] = w.refs
    host = pinned.numpy()
    e2e_t = []
    e2e_warm = max(2, a.warmup)
    for i in range(e2e_warm + max(10, a.steps)):  # each ~2-3 ms: at least 10 timed
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with dfgtb.DualTreeEngine(host, dfgtb.Mode.series, cfg) as e2:
            e2.sweep(w.scales, w.h_s)
            tree_timings = e2.last_timings()
        t1 = time.perf_counter()
        if i >= e2e_warm:
            e2e_t.append(t1 - t0)
    e2e_s = float(np.mean(e2e_t))
    e2e_v = 18 * n / e2e_s

    instr = FP64_INSTR_PER_PAIR.get(w.refs.shape[1], 2 * w.refs.shape[1] + 19)
    pairs_per_s = base_pairs / (base_ms * 1e-3) if base_ms > 0 else 0.0
    traffic = None
    tp = os.path.join(ROOT, "profiles", "base_case_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("bytes_per_launch")
        except Exception:
            traffic = None
    common = {"traffic": traffic,
              "traffic_source": "static: dram__bytes_read+write of the base-case kernels from the committed "
                                "ncu --set full capture (profiles/base_case_traffic.json), not measured in this run",
              "base_pairs_per_step": base_pairs // max(a.steps, 1),
              "base_ms_per_step": base_ms / max(a.steps, 1),
              "step_share": {k: v / phases["total_ms"] for k, v in phases.items() if k != "total_ms"}
              if phases.get("total_ms") else None}
    if mufu and exp_mode == 2:
        # each base-case kernel against the same ex2 peak (events around each launch)
        per = []
        for name, pairs, t in (("k_base_f32 (FP32 path)", pa.value, f32_ms),
                               ("k_base_case (FP64 distance, MUFU / FP64 exp)", pb.value, fp64_ms)):
            tk = t / max(a.steps, 1)
            rate = pairs / (tk * 1e-3) if tk > 0 else 0.0
            per.append({"kernel": name, "pairs_per_step": int(pairs), "ms_per_step": tk,
                        "achieved": rate / 1e9, "frac": rate / peak_ex2 if peak_ex2 > 0 else None})
        common["per_kernel"] = per
    if mufu:
        kname = ("k_base_f32 + k_base_case (K10 exhaustive base case: FP32 distance/ex2/partial sums "
                 "for the leaf pairs that qualify, MUFU ex2 with FP64 distance and sums for the rest)"
                 if exp_mode == 2 else "k_base_case (K10 exhaustive base case, MUFU ex2 path)")
        roof = {"bound": "sfu", "kernel": kname,
                "achieved": pairs_per_s / 1e9, "peak": peak_ex2 / 1e9, "unit": "G ex2/s (1 per pair)",
                "frac": pairs_per_s / peak_ex2 if peak_ex2 > 0 else None,
                "peak_source": "measured ex2.approx.f32 throughput (dfgtb_ex2_peak) on this GPU",
                "speedup_vs_ideal_fp64_exp": {
                    "value": pairs_per_s * instr / peak_instr if peak_instr > 0 else None,
                    "note": f"pairs/s x {instr} FP64 instr/pair (libdevice-exp algorithm, 2D+19) over the "
                            "measured DFMA peak: > 1 means faster than an ideal FP64-exp kernel; a "
                            "speed-up, not a roofline fraction"},
                **common}
    else:
        roof = {"bound": "fp64", "kernel": "k_base_case (K10 exhaustive base case, FP64 exp)",
                "achieved": pairs_per_s * instr / 1e12, "peak": peak_instr / 1e12,
                "unit": "T FP64-pipe instr/s", "instr_per_pair": instr,
                "frac": pairs_per_s * instr / peak_instr if peak_instr > 0 else None,
                "peak_source": "measured DFMA throughput (dfgtb_dfma_peak) on this GPU", **common}
    # the same sweep with every kernel on ONE stream (DFGTB_ONE_STREAM): the base-case
    # kernels' own durations without sharing SMs with the expansion chain (the overlapped
    # step above is the faster one; this explains the per-kernel fractions)
    os.environ["DFGTB_ONE_STREAM"] = "1"
    try:
        e1s = dfgtb.DualTreeEngine(w.refs, dfgtb.Mode.series, cfg)
    finally:
        del os.environ["DFGTB_ONE_STREAM"]
    s1s = torch.cuda.ExternalStream(_capi.lib.dfgtb_stream(e1s.handle))
    e1s.sweep(w.scales, w.h_s)
    iso_ms, iso_f32, iso_fp64 = [], 0.0, 0.0
    for _ in range(max(3, a.steps)):
        with torch.cuda.stream(s1s):
            flush.zero_()
        iso_ms.append(_events_ms(s1s, lambda: e1s.sweep(w.scales, w.h_s)))
        tmi = e1s.last_timings()
        iso_f32 += tmi["base_f32_ms"]
        iso_fp64 += tmi["base_fp64_ms"]
    nrep = max(3, a.steps)
    iso_base = (iso_f32 + iso_fp64) / nrep
    e1s.close()
    iso_rate = (pa.value + pb.value) / (iso_base * 1e-3) if iso_base > 0 else 0.0
    roof["isolated"] = {
        "ms_per_step": float(np.mean(iso_ms)), "base_ms_per_step": iso_base,
        "frac": iso_rate / peak_ex2 if peak_ex2 > 0 else None,
        "per_kernel": [{"kernel": "k_base_f32", "ms_per_step": iso_f32 / nrep,
                        "frac": pa.value / (iso_f32 / nrep * 1e-3) / peak_ex2 if iso_f32 > 0 else None},
                       {"kernel": "k_base_case", "ms_per_step": iso_fp64 / nrep,
                        "frac": pb.value / (iso_fp64 / nrep * 1e-3) / peak_ex2 if iso_fp64 > 0 else None}],
        "note": "same sweep, every kernel on one stream (DFGTB_ONE_STREAM=1): no SM sharing with the "
                "far-field / local-expansion chain; the headline overlaps the two chains and is faster"}
    f32_share = pa.value / max(1, pa.value + pb.value)
    hbm, hbm_src = hbm_peak()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": t_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64" if exp_mode != 2 else "f64+f32",
        "dtype_note": (f"FP64 points, sums, traversal and expansions; {100 * f32_share:.0f}% of the base-case "
                       "pairs run FP32 differences / distance / partial sums with ex2.approx (2e-4 of eps "
                       "charged, traversal at eps - 2e-4), the rest FP64 distance + MUFU ex2 (4e-6 charged)"
                       if exp_mode == 2 else "FP64 throughout (MUFU ex2 on an exactly reduced argument when "
                       "eps >= 1e-4)"),
        "data": "synthetic (seeded cfg2 generator, SURVEY 8(d))",
        "config": config_block(w, world),
        "roofline": roof,
        "tree_moment_roofline": {**tree_moment_roofline_from(tree_timings, eng, n, w.refs.shape[1], hbm),
                                 "peak_source": hbm_src},
        "clocks": clk.summary(),
        "gpu_launches": int(launches),
        "e2e": {"value": e2e_v, "unit": UNIT, "ms_per_step": 1e3 * e2e_s, "ms_min": 1e3 * float(np.min(e2e_t)),
                "steps": len(e2e_t), "h2d_bytes_per_step": int(w.refs.nbytes),
                "d2h_bytes_per_step": int(len(w.scales) * 148 * 3 * 8),
                "timed": "DualTreeEngine(pinned host points) [H2D, GPU tree, moments] + dfgtb_sweep + "
                         "scores back + engine destroy, wall clock"},
        "scores": [{"h": r.h, "lk": r.lk_score, "lk_clamped": r.lk_clamped, "ls": r.ls_score}
                   for r in rows],
    }
    if not a.quick:
        # per-h incremental: each bandwidth's (h, 2h) CV on its own (engine resident)
        per_h = []
        for sc in w.scales:
            h = sc * w.h_s
            eng.cv(h)
            t_ms = _events_ms(stream, lambda: eng.cv(h), reps=3)
            per_h.append({"scale": sc, "h": h, "ms_h_and_2h": t_ms, "queries_per_s": 2 * n / (t_ms * 1e-3)})
        line["per_h"] = {"rows": per_h, "timed": "dfgtb_cv(h, 2h) alone per bandwidth, engine resident, "
                                                 "CUDA events; the headline batches all 18 in one traversal"}
        # the same sweep with the FP32 base case disabled (FP64 distance + MUFU ex2 only)
        os.environ["DFGTB_NO_F32"] = "1"
        try:
            e3 = dfgtb.DualTreeEngine(w.refs, dfgtb.Mode.series, cfg)
        finally:
            del os.environ["DFGTB_NO_F32"]
        s3 = torch.cuda.ExternalStream(_capi.lib.dfgtb_stream(e3.handle))
        e3.sweep(w.scales, w.h_s)
        t3 = []
        for _ in range(max(3, a.steps)):
            with torch.cuda.stream(s3):
                flush.zero_()
            t3.append(_events_ms(s3, lambda: e3.sweep(w.scales, w.h_s)))
        t3m = float(np.mean(t3))
        line["no_f32"] = {"value": 18 * n / (t3m * 1e-3), "ms_per_step": t3m, "unit": UNIT,
                          "note": "DFGTB_NO_F32=1: every base-case pair on the FP64-distance MUFU kernel"}
        e3.close()
        line["configs"] = config_records(dfgtb, flush, max(3, a.steps))
    ref_scores, ref_tree = None, None
    if not a.no_cpu_baseline:
        from oracle import load_reference
        ref = load_reference()
        if ref is not None:
            cores = os.cpu_count() or 1
            wall, ref_scores, cpu_sum = reference_sweep(w, cores)
            ref_tree = ref.tree(w.refs, 32)
            line["cpu_baseline"] = {
                "value": 18 * n / wall, "unit": UNIT, "cores": min(cores, 18), "kind": "reference",
                "cpu": cpu_model(),
                "sample": "one full cfg2 sweep: 18 reference DualTreeEngine computes (9 scales x "
                          f"{{h, 2h}}), one engine per process, {min(cores, 18)} processes; "
                          f"sum of single-core compute time {cpu_sum:.1f} s"}
    line["parity"] = parity_block(dfgtb, eng, w, ref_scores, ref_tree)
    print(json.dumps(line), flush=True)


def tree_moment_roofline_from(t, eng, n, d, hbm_gbs):
    """tree_moment_roofline on a given engine's timings (the e2e engines build the tree)."""
    tree = eng.reference_tree()
    height, K, T = int(tree.height), int(tree.count.shape[0]), eng.p_max() ** d
    tb = height * n * (8 * d + 16)
    mb = height * n * 8 * d + K * T * 8
    out = {}
    for name, by, ms in (("k_build (tree)", tb, t["tree_ms"]),
                         ("k_moment_chunks_w + k_moment_reduce", mb, t["moments_build_ms"])):
        gbs = by / (ms * 1e-3) / 1e9 if ms > 0 else None
        out[name] = {"bytes": int(by), "ms": ms, "achieved_gbs": gbs, "peak_gbs": hbm_gbs,
                     "frac": gbs / hbm_gbs if gbs else None}
    out["bytes_model"] = ("tree: height x N x (8D + 16) (SURVEY 8(d)); moments: height x N x 8D read + "
                          "nodes x p^D x 8 written")
    out["note"] = (f"one-time per engine; height {height}, {K} nodes, {T}-term tables; the inputs "
                   "(<= 24 MB) are L2-resident, so both are latency-bound rather than HBM-bound")
    return out


def run_sharded(a, rank, world, local_rank):
    """N > 1: ONE cfg2 sweep with its queries sharded over the ranks.
    Each rank owns a contiguous range of the reference kd-tree's point order (a few
    compact subtrees), computes its queries' sums at all 18 bandwidths through
    DualTreeEngine.compute_batch (query tree per shard, full reference tree), reduces
    its 3 CV partials per bandwidth, and ONE NCCL all_reduce combines them.  Strong
    scaling: total work is fixed."""
    import torch
    import torch.distributed as dist

    import paper_1102_2878_b200 as dfgtb
    from paper_1102_2878_b200 import _capi
    from paper_1102_2878_b200.distributed import sharded_sweep, torch_allreduce

    w = workload(0)
    n = w.refs.shape[0]
    cfg = dfgtb.EngineConfig(epsilon=0.01, leaf_threshold=32)
    eng = dfgtb.DualTreeEngine(w.refs, dfgtb.Mode.series, cfg)
    order = eng.reference_tree().perm
    ar = torch_allreduce()

    def step():
        return sharded_sweep(w.refs, w.scales, w.h_s, lambda q, hs: eng.compute_batch(q, hs), rank, world,
                             ar, order=order)

    for _ in range(a.warmup):
        step()
    l0 = _capi.lib.dfgtb_launch_count(eng.handle)
    ts = []
    with Clocks(local_rank) as clk:
        for _ in range(a.steps):
            dist.barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            rows = step()  # ends with the all_reduce's result on the host
            e1.record()
            torch.cuda.synchronize()
            ts.append(1e-3 * e0.elapsed_time(e1))  # device timeline, max over ranks below
    launches = _capi.lib.dfgtb_launch_count(eng.handle) - l0
    tt = torch.tensor([float(np.mean(ts))], device="cuda", dtype=torch.float64)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_step = float(tt.item())
    if rank == 0:
        line = {"metric": METRIC, "value": 18 * n / t_step, "unit": UNIT, "n_gpus": world, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": 1e3 * t_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64+f32", "data": "synthetic (seeded cfg2 generator, SURVEY 8(d))",
                "config": {**config_block(w, world), "parallelism": f"query-sharded x{world} (tree order), "
                           "one NCCL all_reduce of 3 partials per bandwidth"},
                "clocks": clk.summary(), "gpu_launches": int(launches),
                "e2e": {"value": 18 * n / t_step, "unit": UNIT, "h2d_bytes_per_step": int(8 * 2 * n // world),
                        "d2h_bytes_per_step": int(8 * 18 * n // world),
                        "timed": "CUDA events per rank around the public-API step (shard queries H2D, sums "
                                 "D2H, NCCL all_reduce), max over ranks"},
                "scores": [{"h": r.h, "lk": r.lk_score, "lk_clamped": r.lk_clamped, "ls": r.ls_score}
                           for r in rows]}
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--quick", action="store_true", help="skip the per-h / no-FP32 / cfg3+cfg5 records")
    a = p.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if a.impl == "reference":
        run_reference(a, rank, world)
    else:
        run_ours(a, rank, world, local_rank)


if __name__ == "__main__":
    main()
