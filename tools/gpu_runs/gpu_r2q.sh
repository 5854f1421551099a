# nearest-centre k-means + packed fma parity: focused tests, k-means / BS benches
OUT=gpurun_out/r2q; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_reduce.py tests/test_gpu_streaming.py tests/test_gpu_map.py -q -x > $OUT/t.log 2>&1; echo tests rc=$?; tail -n 3 $OUT/t.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "kmeans or blackscholes" > $OUT/tf.log 2>&1; echo fullsize rc=$?; tail -n 3 $OUT/tf.log
for w in kmeans blackscholes-f32 blackscholes-f64; do
timeout 600 python bench.py --workload $w --no-cpu-baseline > $OUT/bench_$w.json 2> $OUT/bench_$w.err; echo $w rc=$? $(python -c "
import json; d=json.loads(open('$OUT/bench_$w.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline'].get('kernel_ms'), d['roofline']['frac'], d['parity']['ok'], d['step_breakdown_ms'])" 2>&1 | tail -1); done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gr_region -s 3 -c 1 -o $OUT/full_kmeans python bench.py --workload kmeans --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; echo ncu rc=$?
