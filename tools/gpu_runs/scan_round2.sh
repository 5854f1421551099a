mkdir -p gpurun_out/s2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s2/build.log 2>&1
GRUMPY_SCAN_TMA=1 timeout 600 python -m pytest -q -x tests/test_gpu_scan_slices.py -m gpu > gpurun_out/s2/pytest.log 2>&1; echo pytest rc=$? >> gpurun_out/s2/pytest.log
for lag in 1 2 3; do
GRUMPY_SCAN_TMA=1 GRUMPY_SCAN_LAG=$lag GRUMPY_SCAN_DEFINES=GR_SCAN_STATS timeout 300 python bench.py --workload cumsum --steps 3 --warmup 3 > gpurun_out/s2/stats_l$lag.txt 2>&1
GRUMPY_SCAN_TMA=1 GRUMPY_SCAN_LAG=$lag timeout 300 python bench.py --workload cumsum --steps 20 --warmup 5 > gpurun_out/s2/bench_l$lag.json 2>&1
done
