# k-means: exact fallback out of line (32 regs, full occupancy)
OUT=gpurun_out/r3d; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_reduce.py -q -x > $OUT/t.log 2>&1; echo tests rc=$?; tail -n 2 $OUT/t.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -k kmeans > $OUT/tf.log 2>&1; echo fullsize rc=$?; tail -n 2 $OUT/tf.log
for mb in 0 12; do GRUMPY_NEAREST_MINB=$mb timeout 600 python bench.py --workload kmeans --steps 10 --no-cpu-baseline --e2e-steps 1 > $OUT/km_$mb.json 2> $OUT/km_$mb.err; echo km minb=$mb $(python -c "
import json; d=json.loads(open('$OUT/km_$mb.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['parity']['ok'])" 2>&1 | tail -1); done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gr_region -s 3 -c 1 -o $OUT/full_kmeans python bench.py --workload kmeans --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; echo ncu rc=$?
