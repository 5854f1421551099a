mkdir -p gpurun_out/sg3
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sg3/build.log 2>&1
timeout 900 python -m pytest -q -x tests/test_gpu_scan_slices.py tests/test_gpu_streaming.py tests/test_gpu_fullsize.py -m gpu > gpurun_out/sg3/pytest.log 2>&1; echo pytest rc=$? >> gpurun_out/sg3/pytest.log
timeout 300 python bench.py --workload cumsum --no-cpu-baseline > gpurun_out/sg3/bench_cumsum.json 2>&1
