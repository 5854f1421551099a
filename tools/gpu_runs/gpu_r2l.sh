python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for mb in 0 6 7 8; do
GRUMPY_ROWS_MINB=$mb timeout 600 python bench.py --workload kmeans --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_kmmb_$mb.json 2> gpurun_out/b_kmmb_$mb.err; echo km minb=$mb rc=$? $(python -c "
import json; d=json.loads(open('gpurun_out/b_kmmb_$mb.json').read().strip().splitlines()[-1]); print(d['roofline']['kernel_ms'], d['roofline']['compute']['frac'], d['parity']['ok'], d['parity']['label_mismatches'])" 2>&1 | tail -1); done
