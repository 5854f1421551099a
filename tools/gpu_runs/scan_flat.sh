# flat (axis=None) scans of n-D operands on the TMA path
mkdir -p gpurun_out/fl
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fl/build.log 2>&1
timeout 300 python -m pytest -q -x tests/test_gpu_scan_slices.py -m gpu -k "flat_nd" > gpurun_out/fl/pytest_q.log 2>&1; echo pytest rc=$? >> gpurun_out/fl/pytest_q.log
if grep -q "pytest rc=0" gpurun_out/fl/pytest_q.log; then
  timeout 900 python -m pytest -q -x tests/test_gpu_scan_slices.py tests/test_gpu_streaming.py tests/test_gpu_fullsize.py -m gpu > gpurun_out/fl/pytest.log 2>&1; echo pytest rc=$? >> gpurun_out/fl/pytest.log
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fl/probe.csv python tools/scan_rows_probe.py > gpurun_out/fl/probe.txt 2>&1
fi
