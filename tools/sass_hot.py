#!/usr/bin/env python
"""Summarise an ncu source page (SASS view): instruction mix and the hottest address
ranges by executed warp instructions and by stall samples.

  ncu -i X.ncu-rep --page source --csv --print-source sass > X.csv
  python tools/sass_hot.py X.csv [top]
"""
import csv
import sys
from collections import Counter


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    hdr = next(r for r in rows if len(r) > 2 and r[0] == "Address")
    data = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r[0].startswith("0x")]
    ie = lambda r: float(r["Instructions Executed"] or 0)  # noqa: E731
    ss = lambda r: float(r["Warp Stall Sampling (All Samples)"] or 0)  # noqa: E731
    tot, tots = sum(map(ie, data)), sum(map(ss, data))
    print(f"warp instructions {tot:.4g}, stall samples {tots:.4g}")
    mix = Counter()
    for r in data:
        op = r["Source"].split()[0] if r["Source"].split() else "?"
        if op.startswith("@"):
            op = r["Source"].split()[1]
        mix[op.split(".")[0]] += ie(r)
    print("mix:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in mix.most_common(20)))
    # contiguous blocks of 16 instructions
    blocks = {}
    for i, r in enumerate(data):
        b = i // 16
        e = blocks.setdefault(b, [0.0, 0.0, i])
        e[0] += ie(r)
        e[1] += ss(r)
    print("hottest 16-instruction blocks (index: %instr %stall first-op):")
    for b, (v, s, i) in sorted(blocks.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"  {i:6d}: {100 * v / tot:5.1f}% {100 * s / max(tots, 1):5.1f}%  {data[i]['Source'].strip()[:60]}")


if __name__ == "__main__":
    main()
