#!/bin/bash
# One GPU pass that refreshes the committed evidence: GPU tests, every bench
# workload (JSON lines), per-launch ncu times + DRAM bytes, and one --set full
# capture of the headline kernel.  Output under gpurun_out/round/.
OUT=gpurun_out/round
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for w in blackscholes-f32 blackscholes-f64 listing1 rownorm rownorm-y mlp kmeans jacobi cumsum; do
  timeout 400 python bench.py --workload $w > $OUT/bench_$w.json 2> $OUT/bench_$w.err
done
timeout 300 python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/bench_reference.err
for w in blackscholes-f32 blackscholes-f64 listing1 rownorm rownorm-y mlp kmeans jacobi cumsum; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:gr_ -c 40 --csv --log-file $OUT/launches_$w.csv \
    python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gr_region -s 3 -c 1 \
  -o $OUT/full_blackscholes-f32 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gr_region -s 3 -c 1 \
  -o $OUT/full_kmeans python bench.py --workload kmeans --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gr_region -s 3 -c 1 \
  -o $OUT/full_cumsum python bench.py --workload cumsum --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
echo done
