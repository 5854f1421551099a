# k-means: final fold of per-CTA histogram partials (batched loads) vs grid size and occupancy
OUT=gpurun_out/r3e; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for cfg in "0 2368" "0 592" "0 1184" "12 2368" "12 592"; do set -- $cfg
GRUMPY_NEAREST_MINB=$1 GRUMPY_KEYED_MAX_GRID=$2 timeout 600 python bench.py --workload kmeans --steps 10 --no-cpu-baseline --e2e-steps 1 > $OUT/km_$1_$2.json 2> $OUT/km_$1_$2.err; echo km minb=$1 grid=$2 $(python -c "
import json; d=json.loads(open('$OUT/km_$1_$2.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['parity']['ok'])" 2>&1 | tail -1); done
