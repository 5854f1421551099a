# k-means nearest: register-cap sweep; BS f32: spill-tolerant tuning sweep
OUT=gpurun_out/r2r; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_reduce.py -q -x -k "kmeans or nearest" > $OUT/t.log 2>&1; echo tests rc=$?; tail -n 2 $OUT/t.log
for mb in 0 8 10 12; do GRUMPY_NEAREST_MINB=$mb timeout 600 python bench.py --workload kmeans --steps 10 --no-cpu-baseline --e2e-steps 1 > $OUT/km_$mb.json 2> $OUT/km_$mb.err; echo km minb=$mb $(python -c "
import json; d=json.loads(open('$OUT/km_$mb.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['parity']['ok'], d['step_breakdown_ms']['per_launch'])" 2>&1 | tail -1); done
for tl in 0 8 16; do GRUMPY_TUNE_MAX_LOCAL=$tl timeout 600 python bench.py --steps 10 --no-cpu-baseline --e2e-steps 1 > $OUT/bs_$tl.json 2> $OUT/bs_$tl.err; echo bs tl=$tl $(python -c "
import json; d=json.loads(open('$OUT/bs_$tl.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['roofline']['frac'], d['parity']['ok'])" 2>&1 | tail -1); done
