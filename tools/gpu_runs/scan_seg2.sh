# segmented register-staged scans (line lengths not whole tiles); e2e variance check
mkdir -p gpurun_out/sg2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sg2/build.log 2>&1
timeout 300 python -m pytest -q -x tests/test_gpu_scan_slices.py -m gpu -k segmented > gpurun_out/sg2/pytest_seg.log 2>&1; echo pytest rc=$? >> gpurun_out/sg2/pytest_seg.log
if grep -q "pytest rc=0" gpurun_out/sg2/pytest_seg.log; then
  timeout 400 python -m pytest -q -x tests/test_gpu_scan_slices.py tests/test_gpu_streaming.py -m gpu > gpurun_out/sg2/pytest.log 2>&1; echo pytest rc=$? >> gpurun_out/sg2/pytest.log
fi
for i in 1 2; do
  timeout 300 python bench.py --workload mlp --no-cpu-baseline > gpurun_out/sg2/mlp_$i.json 2>&1
  timeout 300 python bench.py --workload cumsum-rows --no-cpu-baseline > gpurun_out/sg2/cr_$i.json 2>&1
done
