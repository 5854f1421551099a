# TMA scan mailboxes as mbarriers: tests, bench, racecheck of the scan family
mkdir -p gpurun_out/mb
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/mb/build.log 2>&1
timeout 300 python -m pytest -q -x tests/test_gpu_scan_slices.py -m gpu -k "tma_matches or segmented or flat" > gpurun_out/mb/pytest_q.log 2>&1; echo pytest rc=$? >> gpurun_out/mb/pytest_q.log
if grep -q "pytest rc=0" gpurun_out/mb/pytest_q.log; then
  timeout 900 python -m pytest -q -x tests/test_gpu_scan_slices.py tests/test_gpu_streaming.py tests/test_gpu_fullsize.py -m gpu > gpurun_out/mb/pytest.log 2>&1; echo pytest rc=$? >> gpurun_out/mb/pytest.log
  timeout 300 python bench.py --workload cumsum --no-cpu-baseline > gpurun_out/mb/bench_cumsum.json 2>&1
  for tool in memcheck racecheck synccheck; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_check.py scan > gpurun_out/mb/$tool.log 2>&1
    echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/mb/$tool.log | tail -1)" >> gpurun_out/mb/summary.txt
  done
fi
