# BS f32 with ptxas contraction + packed tail; TMA scan without look-back (floor); inexact position test
OUT=gpurun_out/r2w; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_map.py tests/test_gpu_streaming.py -q -x > $OUT/t.log 2>&1; echo tests rc=$?; tail -n 3 $OUT/t.log
timeout 600 python bench.py --steps 20 --no-cpu-baseline --e2e-steps 1 > $OUT/bs.json 2> $OUT/bs.err; echo bs $(python -c "
import json; d=json.loads(open('$OUT/bs.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['roofline']['frac'], d['parity']['ok'], d['parity'].get('max_err'))" 2>&1 | tail -1)
for st in 4 6; do GRUMPY_SCAN_DEFINES=GR_SCAN_NOLB GRUMPY_SCAN_STAGES=$st timeout 600 python bench.py --workload cumsum --steps 10 --no-cpu-baseline --e2e-steps 1 > $OUT/cs_nolb_$st.json 2> $OUT/cs_nolb_$st.err; echo cumsum nolb stages=$st $(python -c "
import json; d=json.loads(open('$OUT/cs_nolb_$st.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['roofline']['frac'])" 2>&1 | tail -1); done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gr_region -s 3 -c 1 -o $OUT/full_cumsum python bench.py --workload cumsum --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; echo ncu rc=$?
