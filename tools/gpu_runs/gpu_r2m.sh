python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python bench.py --gpus 4 --workload rownorm --steps 5 > gpurun_out/mg_rownorm4.json 2> gpurun_out/mg_rownorm4.err; echo rownorm4 rc=$?
timeout 900 python bench.py --gpus 2 --steps 5 > gpurun_out/mg_bs2.json 2> gpurun_out/mg_bs2.err; echo bs2 rc=$?
timeout 900 python bench.py --gpus 2 --workload kmeans --steps 5 > gpurun_out/mg_km2.json 2> gpurun_out/mg_km2.err; echo km2 rc=$?
timeout 900 python bench.py --gpus 2 --impl reference --steps 2 > gpurun_out/mg_ref2.json 2> gpurun_out/mg_ref2.err; echo ref2 rc=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
for f in mg_rownorm4 mg_bs2 mg_km2 mg_ref2; do python -c "
import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', d['n_gpus'], d['value'], d.get('parity',{}).get('ok'), d.get('comm'), d.get('step_breakdown_ms'), d['config'])" 2>&1 | tail -1; done
