#!/usr/bin/env python
"""Group an ncu SASS source page (--page source --csv --print-source sass) into runs of
instructions with equal execution counts (basic blocks) and print the heaviest, with
their opcode mix and stall reasons.

  python tools/sass_blocks.py X.csv [top]
"""
import csv
import sys
from collections import Counter


def op(src):
    t = src.split()
    if not t:
        return "?"
    return (t[1] if t[0].startswith("@") and len(t) > 1 else t[0]).split(".")[0]


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    hdr = next(r for r in rows if len(r) > 2 and r[0] == "Address")
    data = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r[0].startswith("0x")]
    h = len(data) // 2
    if h and len(data) % 2 == 0 and all(data[i]["Source"] == data[h + i]["Source"] for i in range(h)):
        data = data[:h]  # the source page repeats the listing once per profiled pass
    scols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
    blocks, cur = [], None
    for i, r in enumerate(data):
        n = int(float(r["Instructions Executed"] or 0))
        if cur and cur["n"] == n:
            cur["rows"].append(r)
        else:
            cur = {"start": i, "n": n, "rows": [r]}
            blocks.append(cur)
    tot = sum(b["n"] * len(b["rows"]) for b in blocks)
    stot = sum(float(r[c] or 0) for r in data for c in scols)
    print(f"{len(data)} instructions, {tot:.4g} warp instructions executed, {stot:.4g} stall samples")
    for b in sorted(blocks, key=lambda b: -b["n"] * len(b["rows"]))[:top]:
        mix = Counter(op(r["Source"]) for r in b["rows"])
        st = Counter()
        for r in b["rows"]:
            for c in scols:
                st[c.replace("stall_", "")] += float(r[c] or 0)
        ss = sum(st.values())
        print(f"@{b['start']:5d} len {len(b['rows']):4d} x{b['n']:>9d}  {100 * b['n'] * len(b['rows']) / tot:5.1f}% instr "
              f"{100 * ss / max(stot, 1):5.1f}% stalls | {dict(mix.most_common(7))} | "
              f"{ {k: round(100 * v / max(ss, 1)) for k, v in st.most_common(3)} }")


if __name__ == "__main__":
    main()
