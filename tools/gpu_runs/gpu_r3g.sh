OUT=gpurun_out/r3g; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_reduce.py tests/test_gpu_streaming.py tests/test_gpu_distributed.py tests/test_gpu_programs.py -q -x > $OUT/t.log 2>&1; echo tests rc=$?; tail -n 2 $OUT/t.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -k kmeans > $OUT/tf.log 2>&1; echo fullsize rc=$?; tail -n 2 $OUT/tf.log
for rep in 1 2; do timeout 600 python bench.py --workload kmeans --steps 10 --no-cpu-baseline --e2e-steps 1 > $OUT/km$rep.json 2> $OUT/km$rep.err; echo km $(python -c "
import json; d=json.loads(open('$OUT/km$rep.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['roofline']['compute']['frac'], d['parity']['ok'])" 2>&1 | tail -1); done
