#!/usr/bin/env python
"""Benchmark: DFGT kernel-sum queries/sec on BASELINE config 2 (one B200).

Workload (BASELINE.json configs[1]): Q = R = 50,000 points, D = 2,
16-component clipped Gaussian mixture (seeded synthetic), eps = 0.01, leaf 32,
p_max = 6.  One STEP = the full CV bandwidth sweep: 9 bandwidths h = h_s 10^k,
k in {-3,-2,-1,-0.5,0,0.5,1,2,3}, each with kernel sums at h and at 2h (18 sums of
50k queries) and CV_LK + CV_LS reduced on the device.  Metric = queries/sec per h
= 18 * 50,000 / step time (whole job over all ranks).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the reference's own CPU implementation (compiled from
/root/reference into oracle/_ref) on the host cores, same workload.
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
    w = datagen.config(2)
    if rank:  # weak scaling: every rank sweeps its own independent instance
        x = datagen.gauss_mixture_2d(w.refs.shape[0], 1002 + 1000 * rank)
        w = datagen.Workload(w.name, x, None, datagen.silverman_h(x), w.scales)
    return w


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
    from oracle import load_oracle
    hs = [s * w.h_s for s in w.scales]
    jobs = [(w.refs, h, 0.01, 32) for h in hs] + [(w.refs, 2 * h, 0.01, 32) for h in hs]
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(min(cores, len(jobs))) as pool:
        res = pool.map(_ref_one, jobs, chunksize=1)
    wall = time.perf_counter() - t0
    orc = load_oracle()
    n = len(hs)
    scores = []
    for i, h in enumerate(hs):
        lk, cl = orc.lkcv(2, h, res[i][0])
        ls = orc.lscv(2, h, res[i][0], 2 * h, res[n + i][0])
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
                         "sample": "full cfg2 sweep per step: 18 reference DualTreeEngine computes "
                                   "(9 scales x {h, 2h}), one engine per compute, "
                                   f"{min(cores, 18)} processes on the host cores"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def config_block(w, world):
    return {"workload": f"{w.name}: CV sweep 9 x (h, 2h) kernel sums + CV_LK/CV_LS",
            "N": int(w.refs.shape[0]), "D": int(w.refs.shape[1]), "eps": 0.01, "leaf": 32,
            "p_max": 6, "bandwidths": 18, "global_batch": int(18 * w.refs.shape[0] * world),
            "l2": "flushed between timed steps (256 MiB device write)",
            "parallelism": f"replicas{world}" if world > 1 else "single"}


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


def run_ours(a, rank, world, local_rank):
    import torch
    torch.cuda.set_device(local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
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
    if world > 1:
        torch.distributed.barrier()
    l0 = _capi.lib.dfgtb_launch_count(eng.handle)
    ms, base_ms, base_pairs, rows = [], 0.0, 0, None
    f32_ms, fp64_ms = 0.0, 0.0
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
    launches = _capi.lib.dfgtb_launch_count(eng.handle) - l0
    # the base-case pairs on each kernel (every step runs the same sweep)
    ta, tb, pa, pb = C.c_int(), C.c_int(), C.c_uint64(), C.c_uint64()
    _capi.check(_capi.lib.dfgtb_last_base_split(eng.handle, C.byref(ta), C.byref(tb), C.byref(pa), C.byref(pb)))
    torch.cuda.synchronize()
    t_step = float(np.mean(ms))
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([t_step], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step = float(tt.item())
    value = 18 * n * world / (t_step * 1e-3)

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
            r2 = e2.sweep(w.scales, w.h_s)
        t1 = time.perf_counter()
        if i >= e2e_warm:
            e2e_t.append(t1 - t0)
    e2e_s = float(np.mean(e2e_t))
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
    e2e_v = 18 * n * world / e2e_s

    if rank != 0:
        if world > 1:
            torch.distributed.barrier()
            torch.distributed.destroy_process_group()
        return
    instr = FP64_INSTR_PER_PAIR.get(w.refs.shape[1], 2 * w.refs.shape[1] + 19)
    pairs_per_s = base_pairs / (base_ms * 1e-3) if base_ms > 0 else 0.0
    traffic = None
    tp = os.path.join(ROOT, "profiles", "base_case_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("bytes_per_launch")
        except Exception:
            traffic = None
    common = {"traffic": traffic, "base_pairs_per_step": base_pairs // max(a.steps, 1),
              "base_ms_per_step": base_ms / max(a.steps, 1)}
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
        # one MUFU ex2 per (q, r) pair: the SFU pipe is the exp roofline
        kname = ("k_base_f32 + k_base_case (K10 exhaustive base case: FP32 distance/ex2/partial sums "
                 "for the leaf pairs that qualify, MUFU ex2 with FP64 distance and sums for the rest)"
                 if exp_mode == 2 else "k_base_case (K10 exhaustive base case, MUFU ex2 path)")
        roof = {"bound": "sfu", "kernel": kname,
                "achieved": pairs_per_s / 1e9, "peak": peak_ex2 / 1e9, "unit": "G ex2/s (1 per pair)",
                "frac": pairs_per_s / peak_ex2 if peak_ex2 > 0 else None,
                "peak_source": "measured ex2.approx.f32 throughput (dfgtb_ex2_peak) on this GPU",
                "fp64_exp_equivalent": {
                    "frac": pairs_per_s * instr / peak_instr if peak_instr > 0 else None,
                    "note": f"pairs/s x {instr} FP64 instr/pair (libdevice-exp algorithm, 2D+19) "
                            "over the measured DFMA peak: the FP64-exp roofline this path replaces"},
                **common}
    else:
        roof = {"bound": "fp64", "kernel": "k_base_case (K10 exhaustive base case, FP64 exp)",
                "achieved": pairs_per_s * instr / 1e12, "peak": peak_instr / 1e12,
                "unit": "T FP64-pipe instr/s", "instr_per_pair": instr,
                "frac": pairs_per_s * instr / peak_instr if peak_instr > 0 else None,
                "peak_source": "measured DFMA throughput (dfgtb_dfma_peak) on this GPU", **common}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": t_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded cfg2 generator, SURVEY 8(d))",
        "config": config_block(w, world),
        "roofline": roof,
        "clocks": clk.summary(),
        "gpu_launches": int(launches),
        "e2e": {"value": e2e_v, "unit": UNIT, "ms_per_step": 1e3 * e2e_s, "ms_min": 1e3 * float(np.min(e2e_t)),
                "steps": len(e2e_t), "h2d_bytes_per_step": int(w.refs.nbytes),
                "d2h_bytes_per_step": int(len(w.scales) * 148 * 3 * 8)},
        "scores": [{"h": r.h, "lk": r.lk_score, "lk_clamped": r.lk_clamped, "ls": r.ls_score}
                   for r in rows],
    }
    if world == 1 and not a.no_cpu_baseline:
        from oracle import load_reference
        if load_reference() is not None:
            cores = os.cpu_count() or 1
            wall, _, cpu_sum = reference_sweep(w, cores)
            line["cpu_baseline"] = {
                "value": 18 * n / wall, "unit": UNIT, "cores": min(cores, 18), "kind": "reference",
                "sample": "one full cfg2 sweep: 18 reference DualTreeEngine computes (9 scales x "
                          f"{{h, 2h}}), one engine per process, {min(cores, 18)} processes; "
                          f"sum of single-core compute time {cpu_sum:.1f} s"}
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--no-cpu-baseline", action="store_true")
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
