# k-means: two-level fold of the keyed-sum partials; parity + sweep
OUT=gpurun_out/r3f; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_reduce.py tests/test_gpu_streaming.py tests/test_gpu_distributed.py -q -x > $OUT/t.log 2>&1; echo tests rc=$?; tail -n 2 $OUT/t.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -k kmeans > $OUT/tf.log 2>&1; echo fullsize rc=$?; tail -n 2 $OUT/tf.log
for cfg in "0 2368" "0 1184" "12 2368" "8 2368"; do set -- $cfg
GRUMPY_NEAREST_MINB=$1 GRUMPY_KEYED_MAX_GRID=$2 timeout 600 python bench.py --workload kmeans --steps 10 --no-cpu-baseline --e2e-steps 1 > $OUT/km_$1_$2.json 2> $OUT/km_$1_$2.err; echo km minb=$1 grid=$2 $(python -c "
import json; d=json.loads(open('$OUT/km_$1_$2.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['parity']['ok'])" 2>&1 | tail -1); done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gr_region -s 3 -c 1 -o $OUT/full_kmeans python bench.py --workload kmeans --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; echo ncu rc=$?
