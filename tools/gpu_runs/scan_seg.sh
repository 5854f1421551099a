# few long lines along the last axis: the TMA look-back scan with segments
mkdir -p gpurun_out/sg
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sg/build.log 2>&1
timeout 240 python -m pytest -q -x tests/test_gpu_scan_slices.py -m gpu -k segmented > gpurun_out/sg/pytest_seg.log 2>&1; echo pytest rc=$? >> gpurun_out/sg/pytest_seg.log
if grep -q "pytest rc=0" gpurun_out/sg/pytest_seg.log; then
  timeout 400 python -m pytest -q -x tests/test_gpu_scan_slices.py -m gpu > gpurun_out/sg/pytest.log 2>&1; echo pytest rc=$? >> gpurun_out/sg/pytest.log
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sg/probe.csv python tools/scan_rows_probe.py > gpurun_out/sg/probe.txt 2>&1
fi
