# compute-sanitizer over the scan family (TMA ring with the round tree, segments, flat n-D, row scans)
mkdir -p gpurun_out/san
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/san/build.log 2>&1
python tools/sanitize_check.py scan > gpurun_out/san/plain.log 2>&1; echo "plain rc=$?" >> gpurun_out/san/plain.log
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_check.py scan > gpurun_out/san/$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san/$tool.log | tail -1)" >> gpurun_out/san/summary.txt
done
