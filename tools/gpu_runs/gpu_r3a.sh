# warp-per-row ring family, paired + two-pass division: parity (GPU reduce tests under wrow), sweep
OUT=gpurun_out/r3a; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
GRUMPY_ROW_FAMILY=wrow timeout 900 python -m pytest tests/test_gpu_reduce.py -q -x -k "rownorm or sum or softmax" > $OUT/t.log 2>&1; echo wrow tests rc=$?; tail -n 3 $OUT/t.log
for wns in "12,1" "6,2" "8,1" "10,1" "4,3"; do GRUMPY_ROW_FAMILY=wrow GRUMPY_WROW_WNS=$wns timeout 600 python bench.py --workload rownorm --steps 10 --no-cpu-baseline --e2e-steps 1 > $OUT/rn_$wns.json 2> $OUT/rn_$wns.err; echo wrow-pair $wns $(python -c "
import json; d=json.loads(open('$OUT/rn_$wns.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['roofline']['frac'], d['parity'])" 2>&1 | tail -1); done
GRUMPY_ROW_FAMILY=wrow GRUMPY_WROW_WNS=12,1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gr_region -s 3 -c 1 -o $OUT/full_rownorm_wrow python bench.py --workload rownorm --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; echo ncu rc=$?
