python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_all.log 2>&1; echo all rc=$?
for ti in 32 64; do GRUMPY_TILE_TI=$ti timeout 600 python bench.py --workload transpose --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_transpose_$ti.json 2> gpurun_out/b_transpose_$ti.err; echo tr $ti rc=$?; done
GRUMPY_TILE=0 timeout 600 python bench.py --workload transpose --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/b_transpose_off.json 2> gpurun_out/b_transpose_off.err; echo tr off rc=$?
for t in memcheck racecheck; do timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python tools/sanitize_check.py map > gpurun_out/sanitize_${t}_map.log 2>&1; echo "$t map rc=$?"; done
tools/ncu_full.sh transpose transpose_tile
tail -n 2 gpurun_out/gpu_all.log
