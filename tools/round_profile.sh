#!/bin/bash
# One GPU pass that refreshes the committed evidence: GPU tests, every bench
# workload (JSON lines), per-launch ncu times + DRAM bytes, and --set full
# captures of the headline kernels.  Output under gpurun_out/round/.
OUT=gpurun_out/round
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
WL="blackscholes-f32 blackscholes-f64 listing1 rownorm rownorm-y mlp kmeans jacobi cumsum cumsum-rows transpose"
for w in $WL; do
  timeout 600 python bench.py --workload $w > $OUT/bench_$w.json 2> $OUT/bench_$w.err
done
GRUMPY_GEMM_EPILOGUE=0 timeout 600 python bench.py --workload mlp --no-cpu-baseline > $OUT/bench_mlp-noepilogue.json 2> $OUT/bench_mlp-noepilogue.err
timeout 600 python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/bench_reference.err
for w in $WL; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -c 60 --csv --log-file $OUT/launches_$w.csv \
    python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
done
for w in blackscholes-f32 mlp transpose rownorm kmeans cumsum cumsum-rows; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:gr_region -s 3 -c 1 \
    -o $OUT/full_$w python bench.py --workload $w --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/scan_rows_probe.csv \
  python tools/scan_rows_probe.py > $OUT/scan_rows_probe.txt 2>&1
echo done
