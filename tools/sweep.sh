#!/bin/bash
# usage: tools/sweep.sh WORKLOAD "ENV1=a ENV2=b" "ENV1=c" ...   (GPU box)
w=$1; shift
for cfg in "$@"; do
  out=$(env $cfg python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 2>&1 | tail -1)
  echo "$cfg :: $(echo "$out" | python -c 'import json,sys
try:
  d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["ms_per_step"],4), round(r["kernel_ms"],4), round(r["frac"],3))
except Exception as e: print("ERR", e)')"
done
