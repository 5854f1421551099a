mkdir -p gpurun_out/rs
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/rs/build.log 2>&1
timeout 600 python -m pytest -q tests/test_gpu_scan_slices.py -m gpu -k random_shapes > gpurun_out/rs/pytest.log 2>&1; echo pytest rc=$? >> gpurun_out/rs/pytest.log
