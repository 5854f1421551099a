# pageable host arrays through pinned staging slots: streaming tests, e2e (pinned / pageable)
OUT=gpurun_out/r3s; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_streaming.py -q -x > $OUT/t.log 2>&1; echo tests rc=$?; tail -n 2 $OUT/t.log
for w in blackscholes-f32 cumsum rownorm-y kmeans; do timeout 600 python bench.py --workload $w --steps 5 --no-cpu-baseline > $OUT/$w.json 2> $OUT/$w.err; echo $w $(python -c "
import json; d=json.loads(open('$OUT/$w.json').read().strip().splitlines()[-1]); print(d['parity']['ok'], 'e2e', round(d['e2e']['value']/1e9,3), 'pageable', round(d['e2e_pageable']['value']/1e9,3))" 2>&1 | tail -1); done
