# look-back by rounds with the round's aggregates as a warp tree
mkdir -p gpurun_out/tr
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/tr/build.log 2>&1
timeout 400 python -m pytest -q -x tests/test_gpu_scan_slices.py -m gpu -k "tma_matches or segmented or seeded" > gpurun_out/tr/pytest.log 2>&1; echo pytest rc=$? >> gpurun_out/tr/pytest.log
for v in "1 1 2" "1 1 3" "1 2 2" "1 2 3" "0 2 3"; do set -- $v
  GRUMPY_SCAN_TREE=$1 GRUMPY_SCAN_LBW=$2 GRUMPY_SCAN_LAG=$3 timeout 300 python bench.py --workload cumsum --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/tr/t$1_w$2_l$3.json 2>&1
done
GRUMPY_SCAN_LBW=1 GRUMPY_SCAN_LAG=2 GRUMPY_SCAN_DEFINES=GR_SCAN_STATS timeout 300 python bench.py --workload cumsum --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/tr/stats.txt 2>&1
