#!/bin/bash
# Per-launch kernel time + DRAM bytes for every bench workload (run on the GPU
# box; parse with tools/traffic_parse.py).  Numbers printed under ncu are never
# bench values; only the per-launch metrics are used.
mkdir -p gpurun_out/traffic
for w in blackscholes-f32 blackscholes-f64 listing1 rownorm rownorm-y mlp kmeans; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:gr_ -c 40 --csv --log-file gpurun_out/traffic/$w.csv \
    python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
    > gpurun_out/traffic/$w.log 2>&1
  echo "$w rc=$?"
done
