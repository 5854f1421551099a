# look-back fold with batched shared-memory reads: scan tests + cumsum (register-staged and TMA)
OUT=gpurun_out/r3t; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_scan_slices.py tests/test_gpu_streaming.py -q -x > $OUT/t.log 2>&1; echo tests rc=$?; tail -n 2 $OUT/t.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -k cumsum > $OUT/tf.log 2>&1; echo fullsize rc=$?; tail -n 2 $OUT/tf.log
for cfg in "0 6 3 1" "1 6 3 1" "1 6 3 2" "1 6 2 1"; do set -- $cfg
GRUMPY_SCAN_TMA=$1 GRUMPY_SCAN_STAGES=$2 GRUMPY_SCAN_LAG=$3 GRUMPY_SCAN_LBW=$4 timeout 600 python bench.py --workload cumsum --steps 10 --no-cpu-baseline --e2e-steps 1 > $OUT/cs_$1$2$3$4.json 2> $OUT/cs_$1$2$3$4.err; echo cumsum tma=$1 S=$2 lag=$3 lbw=$4 $(python -c "
import json; d=json.loads(open('$OUT/cs_$1$2$3$4.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['roofline']['frac'], d['parity']['ok'])" 2>&1 | tail -1); done
