mkdir -p gpurun_out/fc2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fc2/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_debug.py -m gpu -q -x > gpurun_out/fc2/pytest_debug.log 2>&1; echo pytest rc=$? >> gpurun_out/fc2/pytest_debug.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/fc2/pytest_gpu.log 2>&1; echo pytest rc=$? >> gpurun_out/fc2/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fc2/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/fc2/bench.json 2> gpurun_out/fc2/bench.err
