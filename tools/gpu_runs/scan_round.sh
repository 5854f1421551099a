set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sr/build.log 2>&1
timeout 600 python -m pytest -q -x tests/test_gpu_scan_slices.py -m gpu > gpurun_out/sr/pytest.log 2>&1; echo pytest rc=$?
for v in "1 1" "1 0" "0 1"; do set -- $v
  GRUMPY_SCAN_TMA=$1 GRUMPY_SCAN_ROUND=$2 timeout 300 python bench.py --workload cumsum --steps 20 --warmup 5 > gpurun_out/sr/bench_tma$1_round$2.json 2> gpurun_out/sr/bench_tma$1_round$2.err
done
for lag in 2 4; do GRUMPY_SCAN_TMA=1 GRUMPY_SCAN_LAG=$lag timeout 300 python bench.py --workload cumsum --steps 20 --warmup 5 > gpurun_out/sr/bench_lag$lag.json 2>&1; done
GRUMPY_SCAN_TMA=1 GRUMPY_SCAN_DEFINES=GR_SCAN_NOLB timeout 300 python bench.py --workload cumsum --steps 20 --warmup 5 > gpurun_out/sr/bench_nolb.json 2>&1
