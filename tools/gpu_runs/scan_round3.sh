mkdir -p gpurun_out/s3
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s3/build.log 2>&1
GRUMPY_SCAN_TMA=1 GRUMPY_SCAN_LBW=2 timeout 600 python -m pytest -q -x tests/test_gpu_scan_slices.py -m gpu > gpurun_out/s3/pytest.log 2>&1; echo pytest rc=$? >> gpurun_out/s3/pytest.log
for v in "2 2" "2 3" "3 3" "1 2"; do set -- $v
GRUMPY_SCAN_TMA=1 GRUMPY_SCAN_LBW=$1 GRUMPY_SCAN_LAG=$2 GRUMPY_SCAN_DEFINES=GR_SCAN_STATS timeout 300 python bench.py --workload cumsum --steps 3 --warmup 3 > gpurun_out/s3/stats_w$1_l$2.txt 2>&1
GRUMPY_SCAN_TMA=1 GRUMPY_SCAN_LBW=$1 GRUMPY_SCAN_LAG=$2 timeout 300 python bench.py --workload cumsum --steps 20 --warmup 5 > gpurun_out/s3/bench_w$1_l$2.json 2>&1
done
