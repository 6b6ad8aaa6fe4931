#!/usr/bin/env python
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list.

  python tools/summarize_launches.py LAUNCHES.csv [--last-sweep N_FINALIZE]

Restricts to the measured sweep of tools/profile_step.py (everything after the
warm-up sweep: the launches after the 18th k_finalize) and prints per-kernel
counts, summed device time and share.  ncu serialises launches and runs them
cold, so the SHARES are the meaningful numbers, not the absolute times.
"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    per_sweep = int(sys.argv[2]) if len(sys.argv) > 2 else 18
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    names = [r[ki] for r in data]
    vals = [float(r[mi].replace(",", "")) for r in data]
    fin = [i for i, n in enumerate(names) if "k_finalize" in n]
    start = fin[per_sweep - 1] + 1 if len(fin) >= 2 * per_sweep else 0
    end = fin[2 * per_sweep - 1] + 1 if len(fin) >= 2 * per_sweep else len(names)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, v in zip(names[start:end], vals[start:end]):
        key = n.split("(")[0].replace("dfgtb::<unnamed>::", "").replace("void ", "")[:70]
        agg[key][0] += 1
        agg[key][1] += v
    tot = sum(v for _, v in agg.values())
    print(f"| kernel | launches | device us (cold, serialised) | share |")
    print(f"|---|---:|---:|---:|")
    for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {c} | {v / 1e3:.1f} | {100 * v / tot:.1f}% |")
    print(f"| **total** | {sum(c for c, _ in agg.values())} | {tot / 1e3:.1f} | 100% |")


if __name__ == "__main__":
    main()
