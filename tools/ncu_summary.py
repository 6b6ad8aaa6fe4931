#!/usr/bin/env python
"""Key metrics of an ncu --set full report (first kernel): time, pipes, issue,
occupancy, memory, stall reasons, and the instruction mix from the SASS page.

  python tools/ncu_summary.py REPORT.ncu-rep [--sass]
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r[0], r[1], r[2:]


def main():
    rep = sys.argv[1]
    h, u, vs = raw(rep)
    # --kernel SUBSTR picks the first launch whose name contains it (default: the first)
    want = sys.argv[sys.argv.index("--kernel") + 1] if "--kernel" in sys.argv else None
    v = next((x for x in vs if want is None or want in x[h.index("Kernel Name")]), vs[0])
    print(f"kernel: {v[h.index('Kernel Name')][:100]}")
    for k in KEYS:
        if k in h:
            i = h.index(k)
            print(f"  {k} = {v[i]} {u[i]}")
    st = [(n, v[i]) for i, n in enumerate(h)
          if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")]
    st = sorted(((float(x.replace(",", "")), n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")])
                 for n, x in st), reverse=True)
    print("  stalls/issue: " + ", ".join(f"{n} {x:.2f}" for x, n in st[:8]))
    if "--sass" in sys.argv:
        out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                             capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        hi = [i for i, r in enumerate(rows) if "Instructions Executed" in r][0]
        hd, d = rows[hi], rows[hi + 1:]
        ie, src = hd.index("Instructions Executed"), hd.index("Source")
        ops = collections.Counter()
        for r in d:
            t = r[src].split()
            if not t:
                continue
            op = t[1] if t[0].startswith("@") else t[0]
            ops[op.split(".")[0]] += int(r[ie] or 0)
        tot = sum(ops.values())
        print("  mix: " + ", ".join(f"{k} {100 * c / tot:.1f}%" for k, c in ops.most_common(14)))


if __name__ == "__main__":
    main()
