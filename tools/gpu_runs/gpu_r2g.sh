python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_reduce.py tests/test_gpu_fullsize.py -q -x -k "rownorm or softmax or row" > gpurun_out/coop_tests.log 2>&1; echo tests rc=$?
for pr in 1 0; do for w in rownorm rownorm-y; do GRUMPY_COOP_PAIR=$pr timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_${w}_p$pr.json 2> gpurun_out/b_${w}_p$pr.err; echo $w p$pr rc=$? $(python -c "
import json; d=json.loads(open('gpurun_out/b_${w}_p$pr.json').read().strip().splitlines()[-1]); print(d['roofline']['kernel_ms'], d['roofline']['frac'], d['parity']['ok'], d['parity'].get('total_bitexact'), d['parity'].get('y_bitexact_mismatches'))"); done; done
tools/ncu_full.sh rownorm rownorm_pair
tail -n 3 gpurun_out/coop_tests.log
