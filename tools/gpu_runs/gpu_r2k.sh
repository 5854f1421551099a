python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for cfg in "0 0" "1 0" "1 3" "1 4" "1 5"; do set -- $cfg
GRUMPY_ROWS_DUAL=$1 GRUMPY_ROWS_MINB=$2 timeout 600 python bench.py --workload kmeans --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_km_$1_$2.json 2> gpurun_out/b_km_$1_$2.err; echo km dual=$1 minb=$2 rc=$? $(python -c "
import json; d=json.loads(open('gpurun_out/b_km_$1_$2.json').read().strip().splitlines()[-1]); print(d['roofline']['kernel_ms'], d['roofline']['compute']['frac'], d['parity']['ok'], d['parity']['label_mismatches'])" 2>&1 | tail -1); done
timeout 600 python -m pytest tests/test_gpu_reduce.py tests/test_gpu_programs.py -q -x -k "kmeans or config or argm" > gpurun_out/km_tests.log 2>&1; echo tests rc=$?; tail -n 2 gpurun_out/km_tests.log
