# k-means (vec reuse + f32 shuffles), BS f32 fma-any + spill-tolerant tuning, rownorm coop mode sweep
OUT=gpurun_out/r2t; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_reduce.py tests/test_gpu_streaming.py tests/test_gpu_map.py -q -x > $OUT/t.log 2>&1; echo tests rc=$?; tail -n 2 $OUT/t.log
timeout 600 python bench.py --workload kmeans --steps 10 --no-cpu-baseline --e2e-steps 1 > $OUT/km.json 2> $OUT/km.err; echo km $(python -c "
import json; d=json.loads(open('$OUT/km.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['parity']['ok'])" 2>&1 | tail -1)
for cfg in "any 0" "any 8" "any 16" "one 8"; do set -- $cfg
GRUMPY_FMA_MULTI=$1 GRUMPY_TUNE_MAX_LOCAL=$2 timeout 600 python bench.py --steps 10 --no-cpu-baseline --e2e-steps 1 > $OUT/bs_$1$2.json 2> $OUT/bs_$1$2.err; echo bs fma=$1 tl=$2 $(python -c "
import json; d=json.loads(open('$OUT/bs_$1$2.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['roofline']['frac'], d['parity']['ok'], d['parity'].get('max_err'))" 2>&1 | tail -1); done
for cfg in "plain 2 3" "l2 1 3" "l2 2 3" "l2 4 3" "plain 2 2" "plain 2 4"; do set -- $cfg
GRUMPY_COOP_MODE=$1 GRUMPY_PREFETCH_GROUPS=$2 GRUMPY_COOP_MINBLOCKS=$3 timeout 600 python bench.py --workload rownorm --steps 10 --no-cpu-baseline --e2e-steps 1 > $OUT/rn_$1$2$3.json 2> $OUT/rn_$1$2$3.err; echo rn mode=$1 pg=$2 minb=$3 $(python -c "
import json; d=json.loads(open('$OUT/rn_$1$2$3.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['roofline']['frac'], d['parity']['ok'])" 2>&1 | tail -1); done
