mkdir -p gpurun_out/ob2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ob2/build.log 2>&1
GRUMPY_SCAN_TREE=0 GRUMPY_SCAN_LBW=2 GRUMPY_SCAN_LAG=3 timeout 300 python -m pytest -q -x tests/test_gpu_scan_slices.py -m gpu -k "tma_matches or segmented or seeded" > gpurun_out/ob2/pytest_fold.log 2>&1; echo pytest rc=$? >> gpurun_out/ob2/pytest_fold.log
for mode in "0 2 3" "1 2 2" "1 1 2"; do set -- $mode
  GRUMPY_SCAN_TREE=$1 GRUMPY_SCAN_LBW=$2 GRUMPY_SCAN_LAG=$3 timeout 600 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_check.py scan > gpurun_out/ob2/rc_$1$2.log 2>&1
  echo "tree=$1 lbw=$2 racecheck rc=$? $(grep 'RACECHECK SUMMARY' gpurun_out/ob2/rc_$1$2.log | tail -1)" >> gpurun_out/ob2/summary.txt
done
