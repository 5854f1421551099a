"""Parse tools/traffic_run.sh output into profiles/traffic.json: for each
workload, the DRAM bytes (read + write) per launch of its dominant kernel (the
launch name with the largest total time), as ncu measured them."""
import csv
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def parse(path):
    rows = collections.defaultdict(dict)
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        key = (r["ID"], r["Kernel Name"])
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
                 "msecond": 1e6}.get(unit, 1)
        rows[key][r["Metric Name"]] = v * scale
    return rows


def main(src=os.path.join(ROOT, "gpurun_out", "traffic")):
    out = {}
    detail = {}
    for fn in sorted(os.listdir(src)):
        if not fn.endswith(".csv"):
            continue
        w = fn[:-4]
        rows = parse(os.path.join(src, fn))
        if not rows:
            continue
        # the longest launch is the dominant kernel's (ncu serialises launches)
        (lid, name), m = max(rows.items(), key=lambda kv: kv[1].get("gpu__time_duration.sum", 0))
        traffic = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        out[w] = traffic
        detail[w] = {"launches": len(rows), "dominant_launch_id": lid,
                     "dominant_ns": m.get("gpu__time_duration.sum"), "dram_read": m.get("dram__bytes_read.sum"),
                     "dram_write": m.get("dram__bytes_write.sum")}
    json.dump(out, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
    json.dump(detail, sys.stdout, indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:])
