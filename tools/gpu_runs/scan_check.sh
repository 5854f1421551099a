mkdir -p gpurun_out/sc
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sc/build.log 2>&1
timeout 600 python -m pytest -q -x tests/test_gpu_scan_slices.py tests/test_gpu_streaming.py -m gpu > gpurun_out/sc/pytest.log 2>&1; echo pytest rc=$? >> gpurun_out/sc/pytest.log
