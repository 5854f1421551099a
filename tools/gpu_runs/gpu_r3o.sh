# TMA scan: 64 KB tiles (32 items per thread, two boxes) vs 32 KB
OUT=gpurun_out/r3o; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
GRUMPY_SCAN_TMA=1 GRUMPY_SCAN_ITEMS=32 GRUMPY_SCAN_STAGES=3 timeout 600 python -m pytest tests/test_gpu_scan_slices.py -q -x -k "lookback" > $OUT/t.log 2>&1; echo tests rc=$?; tail -n 2 $OUT/t.log
for cfg in "32 3" "16 6" "32 3 GR_SCAN_NOLB"; do set -- $cfg
GRUMPY_SCAN_DEFINES=$3 GRUMPY_SCAN_TMA=1 GRUMPY_SCAN_ITEMS=$1 GRUMPY_SCAN_STAGES=$2 timeout 600 python bench.py --workload cumsum --steps 10 --no-cpu-baseline --e2e-steps 1 > $OUT/cs_$1_$2_$3.json 2> $OUT/cs_$1_$2_$3.err; echo cumsum items=$1 S=$2 $3 $(python -c "
import json; d=json.loads(open('$OUT/cs_$1_$2_$3.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['roofline']['frac'], d['parity']['ok'])" 2>&1 | tail -1); done
