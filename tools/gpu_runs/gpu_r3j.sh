# rownorm: totals folded per 4096-row block by the completing warp
OUT=gpurun_out/r3j; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_reduce.py tests/test_gpu_distributed.py tests/test_gpu_streaming.py -q -x > $OUT/t.log 2>&1; echo tests rc=$?; tail -n 2 $OUT/t.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -k rownorm > $OUT/tf.log 2>&1; echo fullsize rc=$?; tail -n 2 $OUT/tf.log
for w in rownorm rownorm-y; do for rep in 1 2; do timeout 600 python bench.py --workload $w --steps 20 --no-cpu-baseline --e2e-steps 1 > $OUT/$w$rep.json 2> $OUT/$w$rep.err; echo $w $(python -c "
import json; d=json.loads(open('$OUT/$w$rep.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['roofline']['frac'], d['parity']['ok'], d['parity'].get('total_bitexact'))" 2>&1 | tail -1); done; done
