# debug streamed BS sources; TMA scan with look-back warps + lag: tests, sweep
OUT=gpurun_out/r2y; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python tools/debug_stream_bs.py > $OUT/dbg.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_scan_slices.py -q -x -k "tma or lookback" > $OUT/t.log 2>&1; echo tests rc=$?; tail -n 3 $OUT/t.log
for cfg in "6 3 4" "6 2 4" "6 3 2" "5 2 4"; do set -- $cfg
GRUMPY_SCAN_STAGES=$1 GRUMPY_SCAN_LAG=$2 GRUMPY_SCAN_LBW=$3 timeout 600 python bench.py --workload cumsum --steps 10 --no-cpu-baseline --e2e-steps 1 > $OUT/cs_$1$2$3.json 2> $OUT/cs_$1$2$3.err; echo cumsum S=$1 lag=$2 lbw=$3 $(python -c "
import json; d=json.loads(open('$OUT/cs_$1$2$3.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['roofline']['frac'], d['parity']['ok'])" 2>&1 | tail -1); done
