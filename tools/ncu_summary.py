#!/usr/bin/env python
"""Summarise an ncu report (--set full) into the numbers the roofline cites.

usage: python tools/ncu_summary.py REPORT.ncu-rep [label] >> profiles/<round>_summary.md
Prints one markdown block: duration, DRAM bytes (traffic), DRAM/SM throughput,
issue activity, occupancy, registers, and the dynamic SASS mix per element
when --elements N is given.
"""
import argparse
import collections
import csv
import io
import subprocess

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__cycles_elapsed.avg.per_second", "lts__t_sector_hit_rate.pct",
]


def ncu(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True)
    return list(csv.reader(io.StringIO(out.stdout)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("label", nargs="?", default="")
    ap.add_argument("--elements", type=float, default=0)
    a = ap.parse_args()
    rows = ncu(a.rep, "raw")
    hdr, units, vals = rows[0], rows[1], rows[2]
    print(f"### {a.label or a.rep}\n")
    print("| metric | value | unit |\n|---|---|---|")
    got = {}
    for i, h in enumerate(hdr):
        if h in KEYS:
            got[h] = (vals[i], units[i])
    for k in KEYS:
        if k in got:
            print(f"| {k} | {got[k][0]} | {got[k][1]} |")
    src = ncu(a.rep, "source", ["--print-source", "sass"])
    if len(src) > 2:
        h = src[1]
        ie = h.index("Instructions Executed")
        sc = h.index("Source")
        c = collections.Counter()
        tot = 0
        for r in src[2:]:
            try:
                n = int(r[ie])
            except (ValueError, IndexError):
                continue
            t = r[sc].strip().split()
            op = t[1] if t and t[0].startswith("@") else (t[0] if t else "?")
            c[op.split(".")[0]] += n
            tot += n
        if a.elements:
            print(f"\ndynamic SASS per element: {tot * 32 / a.elements:.1f} thread-instructions; top opcodes: " +
                  ", ".join(f"{k} {v * 32 / a.elements:.1f}" for k, v in c.most_common(12)))
        else:
            print(f"\nwarp instructions executed: {tot}")
    print()


if __name__ == "__main__":
    main()
