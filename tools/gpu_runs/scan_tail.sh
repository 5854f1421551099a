# 1-D scans whose length is not a multiple of a 128-byte line on the TMA path
mkdir -p gpurun_out/st2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/st2/build.log 2>&1
timeout 300 python -m pytest -q -x tests/test_gpu_scan_slices.py -m gpu -k "tma_matches or seeded" > gpurun_out/st2/pytest_tail.log 2>&1; echo pytest rc=$? >> gpurun_out/st2/pytest_tail.log
if grep -q "pytest rc=0" gpurun_out/st2/pytest_tail.log; then
  timeout 600 python -m pytest -q -x tests/test_gpu_scan_slices.py tests/test_gpu_streaming.py tests/test_gpu_fullsize.py -m gpu > gpurun_out/st2/pytest.log 2>&1; echo pytest rc=$? >> gpurun_out/st2/pytest.log
fi
