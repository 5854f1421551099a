"""Summarise an ncu report: SOL, occupancy, issue and the top stall reasons."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "sm__inst_executed.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct"]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    d = {h[i]: (v[i], u[i]) for i in range(len(h))}
    for k in KEYS:
        if k in d:
            print(f"{k:60s} {d[k][0]} {d[k][1]}")
    st = [(k, float(d[k][0].replace(",", "") or 0)) for k in d
          if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
    tot = sum(x for _, x in st) or 1
    for k, x in sorted(st, key=lambda t: -t[1])[:10]:
        print(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {x:8.0f} {100 * x / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
