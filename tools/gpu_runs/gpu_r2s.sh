# k-means: row prefetch / 32-bit match / register cap sweep + read-bandwidth probe
OUT=gpurun_out/r2s; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_reduce.py -q -x > $OUT/t.log 2>&1; echo tests rc=$?; tail -n 2 $OUT/t.log
for cfg in "1 1 10" "0 1 10" "1 0 10" "1 1 8" "1 1 12" "1 1 0"; do set -- $cfg
GRUMPY_ROW_PREFETCH=$1 GRUMPY_MATCH32=$2 GRUMPY_NEAREST_MINB=$3 timeout 600 python bench.py --workload kmeans --steps 10 --no-cpu-baseline --e2e-steps 1 > $OUT/km_$1$2$3.json 2> $OUT/km_$1$2$3.err; echo km pf=$1 m32=$2 minb=$3 $(python -c "
import json; d=json.loads(open('$OUT/km_$1$2$3.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['parity']['ok'])" 2>&1 | tail -1); done
timeout 300 python tools/read_probe.py > $OUT/read_probe.txt 2>&1; cat $OUT/read_probe.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gr_region -s 3 -c 1 -o $OUT/full_kmeans python bench.py --workload kmeans --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; echo ncu rc=$?
