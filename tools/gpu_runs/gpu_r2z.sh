# BS explicit fusion first/last; scan TMA J/R + single look-back warp; wrow two-pass division
OUT=gpurun_out/r2z; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_map.py tests/test_gpu_streaming.py -q -x > $OUT/t.log 2>&1; echo tests rc=$?; tail -n 2 $OUT/t.log
for pk in first last; do GRUMPY_FMA_PICK=$pk timeout 600 python bench.py --steps 20 --no-cpu-baseline --e2e-steps 1 > $OUT/bs_$pk.json 2> $OUT/bs_$pk.err; echo bs pick=$pk $(python -c "
import json; d=json.loads(open('$OUT/bs_$pk.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['roofline']['frac'], d['parity']['ok'], d['parity'].get('max_err'))" 2>&1 | tail -1); done
for cfg in "6 3 1 X" "6 3 2 GR_SCAN_J=4,GR_SCAN_R=4" "6 1 1 X" "6 3 1 GR_SCAN_NOLB"; do set -- $cfg
GRUMPY_SCAN_DEFINES=$([ "$4" = X ] || echo $4) GRUMPY_SCAN_STAGES=$1 GRUMPY_SCAN_LAG=$2 GRUMPY_SCAN_LBW=$3 timeout 600 python bench.py --workload cumsum --steps 10 --no-cpu-baseline --e2e-steps 1 > $OUT/cs_$1$2$3.json 2> $OUT/cs_$1$2$3.err; echo cumsum S=$1 lag=$2 lbw=$3 $4 $(python -c "
import json; d=json.loads(open('$OUT/cs_$1$2$3.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['roofline']['frac'], d['parity']['ok'])" 2>&1 | tail -1); done
for wns in "12,1" "6,2" "8,1"; do GRUMPY_ROW_FAMILY=wrow GRUMPY_WROW_WNS=$wns timeout 600 python bench.py --workload rownorm --steps 10 --no-cpu-baseline --e2e-steps 1 > $OUT/rn_$wns.json 2> $OUT/rn_$wns.err; echo wrow2p $wns $(python -c "
import json; d=json.loads(open('$OUT/rn_$wns.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['roofline']['frac'], d['parity']['ok'])" 2>&1 | tail -1); done
