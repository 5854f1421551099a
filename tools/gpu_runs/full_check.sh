mkdir -p gpurun_out/fc
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fc/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/fc/pytest_gpu.log 2>&1; echo pytest rc=$? >> gpurun_out/fc/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fc/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/fc/bench.json 2> gpurun_out/fc/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/fc/bench_ref.json 2> gpurun_out/fc/bench_ref.err
