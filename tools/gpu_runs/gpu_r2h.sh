python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for vec in 2 4; do for w in rownorm rownorm-y; do GRUMPY_COOP_VEC=$vec timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_${w}_v$vec.json 2> gpurun_out/b_${w}_v$vec.err; echo $w v$vec rc=$? $(python -c "
import json; d=json.loads(open('gpurun_out/b_${w}_v$vec.json').read().strip().splitlines()[-1]); print(d['roofline']['kernel_ms'], d['roofline']['frac'], d['parity']['ok'], d['parity'].get('total_bitexact'), d['parity'].get('y_bitexact_mismatches'))"); done; done
GRUMPY_COOP_VEC=2 tools/ncu_full.sh rownorm rownorm_v2
python tools/ncu_stalls.py gpurun_out/rownorm_v2.ncu-rep | head -8
