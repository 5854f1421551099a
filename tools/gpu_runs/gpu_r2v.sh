# TMA scan with static round-robin tiles (stage sweep) + warp-per-row ring family sweep for rownorm
OUT=gpurun_out/r2v; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_scan_slices.py -q -x -k "tma or lookback" > $OUT/t.log 2>&1; echo tests rc=$?; tail -n 3 $OUT/t.log
for st in 3 4 6; do GRUMPY_SCAN_STAGES=$st timeout 600 python bench.py --workload cumsum --steps 10 --no-cpu-baseline --e2e-steps 1 > $OUT/cs_$st.json 2> $OUT/cs_$st.err; echo cumsum stages=$st $(python -c "
import json; d=json.loads(open('$OUT/cs_$st.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['roofline']['frac'], d['parity']['ok'])" 2>&1 | tail -1); done
for wns in "4,3" "6,2" "12,1" "8,1"; do GRUMPY_ROW_FAMILY=wrow GRUMPY_WROW_WNS=$wns timeout 600 python bench.py --workload rownorm --steps 10 --no-cpu-baseline --e2e-steps 1 > $OUT/rn_$wns.json 2> $OUT/rn_$wns.err; echo wrow $wns $(python -c "
import json; d=json.loads(open('$OUT/rn_$wns.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['roofline']['frac'], d['parity']['ok'])" 2>&1 | tail -1); done
