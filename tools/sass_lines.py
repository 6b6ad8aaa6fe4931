#!/usr/bin/env python
"""Per-source-line instruction and stall-sample shares of one kernel from an ncu report.

  ncu -i REP --page source --csv --print-source sass > k.csv
  nvdisasm -g <cubin> > all.sass            (cuobjdump -xelf all build/execute.o)
  python tools/sass_lines.py k.csv all.sass <mangled-kernel-prefix> <source.cu> [N]
"""
import csv
import re
import sys
from collections import defaultdict


def main():
    csvp, sassp, fn, srcp = sys.argv[1:5]
    top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
    L = open(sassp).read().split("\n")
    start = [i for i, l in enumerate(L) if l.startswith(".text." + fn)][0]
    cur, a2l = None, {}
    for l in L[start + 1:]:
        if l.startswith(".text."):
            break
        m = re.search(r"line (\d+)", l)
        if "//## File" in l and m:
            cur = int(m.group(1))
        m2 = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
        if m2:
            a2l[int(m2.group(1), 16)] = cur
    rows = list(csv.reader(open(csvp)))
    hdr, data = rows[1], [r for r in rows[2:] if r and r[0].startswith("0x")]
    ia = hdr.index("Instructions Executed")
    ss = hdr.index("Warp Stall Sampling (All Samples)")
    base = int(data[0][0], 16)
    byl, bys = defaultdict(int), defaultdict(int)
    tot = sum(int(r[ia] or 0) for r in data)
    tots = sum(int(r[ss] or 0) for r in data)
    mufu = sum(int(r[ia] or 0) for r in data if "MUFU.EX2" in r[1])
    for r in data:
        ln = a2l.get(int(r[0], 16) - base)
        byl[ln] += int(r[ia] or 0)
        bys[ln] += int(r[ss] or 0)
    src = open(srcp).read().split("\n")
    print(f"warp instructions {tot}, MUFU.EX2 {mufu}, stall samples {tots}")
    for ln, v in sorted(byl.items(), key=lambda x: -x[1])[:top]:
        s = src[ln - 1].strip()[:80] if ln else "?"
        print(f"{ln}: inst {v / tot:.3f} stall {bys[ln] / tots:.3f}  {s}")


if __name__ == "__main__":
    main()
