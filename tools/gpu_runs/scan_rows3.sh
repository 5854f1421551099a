# scans along the contiguous axis: lines per warp x chunk width (columns in flight per line)
mkdir -p gpurun_out/sr5
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sr5/build.log 2>&1
for v in "32 64" "16 64" "16 96" "16 128" "8 128" "8 192"; do set -- $v
  GRUMPY_SCAN_ROWS_RPW=$1 GRUMPY_SCAN_ROWS_CW=$2 timeout 600 python bench.py --workload cumsum-rows --steps 10 --warmup 3 --e2e-steps 1 > gpurun_out/sr5/r$1_cw$2.json 2> gpurun_out/sr5/r$1_cw$2.err
done
GRUMPY_SCAN_ROWS_RPW=16 GRUMPY_SCAN_ROWS_CW=96 timeout 900 python -m pytest -q -x tests/test_gpu_scan_slices.py -m gpu -k "rows" > gpurun_out/sr5/pytest.log 2>&1; echo pytest rc=$? >> gpurun_out/sr5/pytest.log
