#!/usr/bin/env python
"""A/B timing of library variants on the bench workload (config-2 sweep, engine
resident): for each libdfgtb.so given, a fresh process times --steps sweeps and prints
ms/step and the per-phase device times.

  python tools/ab.py [--config 2] [--steps 20] lib1.so lib2.so:DFGTB_ONE_STREAM=1 ...
"""
import json
import os
import subprocess
import sys

CHILD = r'''
import os, sys, json, numpy as np
sys.path.insert(0, os.environ["ROOT"])
import torch
import paper_1102_2878_b200 as dfgtb
from paper_1102_2878_b200 import _capi, datagen
k = int(os.environ["CFG"]); steps = int(os.environ["STEPS"])
w = datagen.config(k)
r = w.refs.astype(np.float32) if k == 5 else w.refs
q = w.queries.astype(np.float32) if k == 5 else None
e = dfgtb.DualTreeEngine(r, config=dfgtb.EngineConfig(epsilon=w.epsilons[0], leaf_threshold=32))
st = torch.cuda.ExternalStream(_capi.lib.dfgtb_stream(e.handle))
hs = [s * w.h_s for s in w.scales]
run = (lambda: e.sweep(w.scales, w.h_s)) if q is None else (lambda: e.compute_batch(q, hs))
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for _ in range(3): run()
ms, ph = [], {}
for _ in range(steps):
    with torch.cuda.stream(st): flush.zero_()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st); run(); b.record(st); b.synchronize(); ms.append(a.elapsed_time(b))
    for kk, v in e.last_timings().items(): ph[kk] = ph.get(kk, 0) + v / steps
print(json.dumps({"ms": float(np.mean(ms)), "min": float(np.min(ms)), "med": float(np.median(ms)), "max": float(np.max(ms)), **{kk: round(v, 4) for kk, v in ph.items()}}))
'''


def main():
    args = sys.argv[1:]
    cfg, steps = "2", "20"
    while args and args[0].startswith("--"):
        if args[0] == "--config":
            cfg = args[1]
        elif args[0] == "--steps":
            steps = args[1]
        args = args[2:]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for spec in args:  # lib.so[:VAR=VALUE[,VAR=VALUE..]]
        lib, _, extra = spec.partition(":")
        env = dict(os.environ, DFGTB_LIB=os.path.abspath(lib), ROOT=root, CFG=cfg, STEPS=steps)
        env.update(kv.split("=", 1) for kv in extra.split(",") if kv)
        out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-1500:]
        print(f"{spec}: {line}", flush=True)


if __name__ == "__main__":
    main()
