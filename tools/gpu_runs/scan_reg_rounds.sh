# register-staged long scan with static round-robin tiles + the round tree look-back
mkdir -p gpurun_out/rr
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/rr/build.log 2>&1
timeout 300 python -m pytest -q -x tests/test_gpu_scan_slices.py -m gpu -k "lookback or seeded" > gpurun_out/rr/pytest_q.log 2>&1; echo pytest rc=$? >> gpurun_out/rr/pytest_q.log
if grep -q "pytest rc=0" gpurun_out/rr/pytest_q.log; then
  timeout 900 python -m pytest -q -x tests/test_gpu_scan_slices.py tests/test_gpu_streaming.py tests/test_gpu_fullsize.py -m gpu > gpurun_out/rr/pytest.log 2>&1; echo pytest rc=$? >> gpurun_out/rr/pytest.log
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rr/probe.csv python tools/scan_rows_probe.py > gpurun_out/rr/probe.txt 2>&1
  GRUMPY_SCAN_REG_ROUNDS=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rr/probe_walk.csv python tools/scan_rows_probe.py > gpurun_out/rr/probe_walk.txt 2>&1
fi
