# seeded scans (streamed carry in one pass); streaming + scan tests; cumsum e2e
OUT=gpurun_out/r3r; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_scan_slices.py tests/test_gpu_streaming.py -q -x > $OUT/t.log 2>&1; echo tests rc=$?; tail -n 2 $OUT/t.log
timeout 600 python bench.py --workload cumsum --steps 10 --no-cpu-baseline > $OUT/cs.json 2> $OUT/cs.err; echo cumsum $(python -c "
import json; d=json.loads(open('$OUT/cs.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['parity']['ok'], d['e2e'], d.get('e2e_pageable'))" 2>&1 | tail -1)
