# TMA-fed look-back scan: parity vs register-staged, full size, bench + ncu
OUT=gpurun_out/r2u; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_scan_slices.py -q -x > $OUT/t.log 2>&1; echo tests rc=$?; tail -n 15 $OUT/t.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -k cumsum > $OUT/tf.log 2>&1; echo fullsize rc=$?; tail -n 3 $OUT/tf.log
for st in 6 4 3; do GRUMPY_SCAN_STAGES=$st timeout 600 python bench.py --workload cumsum --steps 10 --no-cpu-baseline --e2e-steps 1 > $OUT/cs_$st.json 2> $OUT/cs_$st.err; echo cumsum stages=$st $(python -c "
import json; d=json.loads(open('$OUT/cs_$st.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['roofline']['frac'], d['parity'])" 2>&1 | tail -1); done
GRUMPY_SCAN_TMA=0 timeout 600 python bench.py --workload cumsum --steps 10 --no-cpu-baseline --e2e-steps 1 > $OUT/cs_old.json 2> $OUT/cs_old.err; echo cumsum old $(python -c "
import json; d=json.loads(open('$OUT/cs_old.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['roofline']['frac'])" 2>&1 | tail -1)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gr_region -s 3 -c 1 -o $OUT/full_cumsum python bench.py --workload cumsum --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; echo ncu rc=$?
