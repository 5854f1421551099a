# several look-back warps hand the CTA prefix over by mbarrier: tests in both modes, racecheck, bench
mkdir -p gpurun_out/ob
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ob/build.log 2>&1
GRUMPY_SCAN_LBW=2 timeout 300 python -m pytest -q -x tests/test_gpu_scan_slices.py -m gpu -k "tma_matches or segmented or seeded or flat or random" > gpurun_out/ob/pytest_lbw2.log 2>&1; echo pytest rc=$? >> gpurun_out/ob/pytest_lbw2.log
GRUMPY_SCAN_TREE=0 GRUMPY_SCAN_LBW=2 GRUMPY_SCAN_LAG=3 timeout 300 python -m pytest -q -x tests/test_gpu_scan_slices.py -m gpu -k "tma_matches or segmented or seeded" > gpurun_out/ob/pytest_fold.log 2>&1; echo pytest rc=$? >> gpurun_out/ob/pytest_fold.log
GRUMPY_SCAN_TREE=0 GRUMPY_SCAN_LBW=2 GRUMPY_SCAN_LAG=3 timeout 600 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_check.py scan > gpurun_out/ob/racecheck_fold.log 2>&1; echo "racecheck rc=$? $(grep 'RACECHECK SUMMARY' gpurun_out/ob/racecheck_fold.log | tail -1)" >> gpurun_out/ob/summary.txt
GRUMPY_SCAN_TREE=0 GRUMPY_SCAN_LBW=2 GRUMPY_SCAN_LAG=3 timeout 300 python bench.py --workload cumsum --no-cpu-baseline --e2e-steps 1 > gpurun_out/ob/bench_fold.json 2>&1
timeout 300 python bench.py --workload cumsum --no-cpu-baseline --e2e-steps 1 > gpurun_out/ob/bench_default.json 2>&1
