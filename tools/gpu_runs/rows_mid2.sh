mkdir -p gpurun_out/rm2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/rm2/build.log 2>&1
timeout 900 python -m pytest -q -x tests/test_gpu_scan_slices.py tests/test_gpu_fullsize.py tests/test_gpu_streaming.py -m gpu > gpurun_out/rm2/pytest.log 2>&1; echo pytest rc=$? >> gpurun_out/rm2/pytest.log
timeout 300 python bench.py --workload cumsum-rows --no-cpu-baseline --e2e-steps 1 > gpurun_out/rm2/bench.json 2>&1
