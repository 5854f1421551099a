python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in 1 0; do GRUMPY_CONTRACT=$c timeout 600 python bench.py --steps 20 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_bs_c$c.json 2> gpurun_out/b_bs_c$c.err; echo bs contract=$c rc=$? $(python -c "
import json; d=json.loads(open('gpurun_out/b_bs_c$c.json').read().strip().splitlines()[-1]); print(d['roofline']['kernel_ms'], d['roofline']['frac'], d['parity'])" 2>&1 | tail -1); done
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_all.log 2>&1; echo all rc=$?; tail -n 2 gpurun_out/gpu_all.log
