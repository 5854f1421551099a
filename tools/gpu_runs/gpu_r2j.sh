python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_all.log 2>&1; echo all rc=$?
timeout 600 python bench.py > gpurun_out/b_default.json 2> gpurun_out/b_default.err; echo default rc=$?
GRUMPY_GEMM_EPILOGUE=0 timeout 600 python bench.py --workload mlp --steps 10 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_mlp_noepi.json 2> gpurun_out/b_mlp_noepi.err; echo noepi rc=$?
for w in kmeans listing1; do timeout 600 python bench.py --workload $w --steps 10 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_$w.json 2> gpurun_out/b_$w.err; echo $w rc=$?; done
tail -n 2 gpurun_out/gpu_all.log
python -c "
import json
for f in ['b_default','b_mlp_noepi','b_kmeans','b_listing1']:
    d=json.loads(open('gpurun_out/'+f+'.json').read().strip().splitlines()[-1]); print(f, d['ms_per_step'], d['roofline']['frac'], d['step_breakdown_ms'], d['parity']['ok'])
"
