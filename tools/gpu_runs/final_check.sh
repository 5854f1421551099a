mkdir -p gpurun_out/final
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/final/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/final/pytest_gpu.log 2>&1; echo pytest rc=$? >> gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err
