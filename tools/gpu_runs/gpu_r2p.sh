# Round-2 re-entry check at HEAD: GPU tests, smoke, default bench, rownorm/kmeans lines
OUT=gpurun_out/r2p; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/gpu_all.log 2>&1; echo all rc=$?; tail -n 2 $OUT/gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo smoke rc=$?
for w in blackscholes-f32 rownorm kmeans cumsum blackscholes-f64; do
timeout 600 python bench.py --workload $w > $OUT/bench_$w.json 2> $OUT/bench_$w.err; echo $w rc=$? $(python -c "
import json; d=json.loads(open('$OUT/bench_$w.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline'].get('kernel_ms'), d['roofline']['frac'], d['parity']['ok'], d['e2e']['value'])" 2>&1 | tail -1); done
