python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for cfg in "plain 256" "plain 128" "tma 128" "tma 64" "async 128"; do set -- $cfg
for w in rownorm rownorm-y; do GRUMPY_COOP_MODE=$1 GRUMPY_COOP_BLOCK=$2 timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_${w}_$1_$2.json 2> gpurun_out/b_${w}_$1_$2.err; echo $w $1 $2 rc=$? $(python -c "
import json; d=json.loads(open('gpurun_out/b_${w}_$1_$2.json').read().strip().splitlines()[-1]); print(d['roofline']['kernel_ms'], d['roofline']['frac'], d['parity']['ok'], d['parity'].get('total_bitexact'), d['parity'].get('y_bitexact_mismatches'))" 2>&1 | tail -1); done; done
