#!/usr/bin/env python
"""Per-kernel roofline table from an ncu metrics CSV of tools/profile_step.py:

  ncu --metrics <METRICS below> --clock-control none --csv --log-file K.csv \\
      python tools/profile_step.py --config 2
  python tools/kernel_table.py K.csv [HBM_GBPS]

Every kernel of the run (engine creation, warm-up sweep, measured sweep), grouped by
name: launches, device time, and the pipe / DRAM utilisation of its time-weighted
launches: FP64 pipe, XU (MUFU) pipe, FMA pipe, issue slots, DRAM GB/s and its fraction
of the measured HBM peak.  ncu serialises and runs every launch cold: the utilisation
figures are per kernel, the absolute times are upper bounds.
"""
import collections
import csv
import sys

METRICS = ["gpu__time_duration.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum",
           "dram__bytes_write.sum"]


def main():
    path = sys.argv[1]
    hbm = float(sys.argv[2]) if len(sys.argv) > 2 else 6526.8
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    launches = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        key = (r[0], r[ki])
        v = float(r[vi].replace(",", "")) if r[vi] not in ("", "n/a") else 0.0
        unit = r[ui]
        if r[mi] == "gpu__time_duration.sum":
            v = v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)  # -> us
        if r[mi].startswith("dram__bytes"):
            v = v * {"byte": 1.0, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "GB": 1e9}.get(unit, 1.0)
        launches.setdefault(key, {})[r[mi]] = v
    agg = collections.OrderedDict()
    for (_, name), m in launches.items():
        short = name.split("(")[0].replace("dfgtb::", "").replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
        g = agg.setdefault(short, {"n": 0, "t": 0.0, "w": collections.Counter(), "bytes": 0.0})
        t = m.get("gpu__time_duration.sum", 0.0)
        g["n"] += 1
        g["t"] += t
        g["bytes"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        for k in METRICS[1:5]:
            g["w"][k] += t * m.get(k, 0.0)
    tot = sum(g["t"] for g in agg.values())
    print("| kernel | launches | device us | share | FP64 pipe % | XU pipe % | FMA pipe % | issue % | DRAM GB/s | % of HBM |")
    print("|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|")
    for k, g in sorted(agg.items(), key=lambda kv: -kv[1]["t"]):
        t = g["t"]
        if t <= 0:
            continue
        w = {m: g["w"][m] / t for m in METRICS[1:5]}
        bw = g["bytes"] / (t * 1e-6) / 1e9
        print(f"| `{k[:48]}` | {g['n']} | {t:.1f} | {100 * t / tot:.1f}% | {w[METRICS[1]]:.1f} | {w[METRICS[2]]:.1f} | "
              f"{w[METRICS[3]]:.1f} | {w[METRICS[4]]:.1f} | {bw:.0f} | {100 * bw / hbm:.1f}% |")
    print(f"| **total** | {sum(g['n'] for g in agg.values())} | {tot:.1f} | 100% | | | | | | |")


if __name__ == "__main__":
    main()
