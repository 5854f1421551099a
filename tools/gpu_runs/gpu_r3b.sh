# BS fusion variants (x2 for noise); scan look-back window geometry (TMA and register-staged); k-means repeat
OUT=gpurun_out/r3b; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for rep in 1 2; do for m in one any; do GRUMPY_FMA_MULTI=$m timeout 600 python bench.py --steps 20 --no-cpu-baseline --e2e-steps 1 > $OUT/bs_$m$rep.json 2> $OUT/bs_$m$rep.err; echo bs multi=$m rep=$rep $(python -c "
import json; d=json.loads(open('$OUT/bs_$m$rep.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['roofline']['frac'], d['parity']['ok'])" 2>&1 | tail -1); done; done
for cfg in "1 GR_SCAN_J=16,GR_SCAN_R=1" "1 GR_SCAN_J=8,GR_SCAN_R=2" "1 GR_SCAN_J=4,GR_SCAN_R=4" "0 GR_SCAN_J=4,GR_SCAN_R=4" "0 GR_SCAN_J=8,GR_SCAN_R=2"; do set -- $cfg
GRUMPY_SCAN_TMA=$1 GRUMPY_SCAN_DEFINES=$2 timeout 600 python bench.py --workload cumsum --steps 10 --no-cpu-baseline --e2e-steps 1 > $OUT/cs_$1_$2.json 2> $OUT/cs_$1_$2.err; echo cumsum tma=$1 $2 $(python -c "
import json; d=json.loads(open('$OUT/cs_$1_$2.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['roofline']['frac'], d['parity']['ok'])" 2>&1 | tail -1); done
timeout 600 python bench.py --workload kmeans --steps 10 --no-cpu-baseline --e2e-steps 1 > $OUT/km.json 2> $OUT/km.err; echo km $(python -c "
import json; d=json.loads(open('$OUT/km.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['parity']['ok'])" 2>&1 | tail -1)
