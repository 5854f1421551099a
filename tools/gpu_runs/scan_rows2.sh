# scans along the contiguous axis: register-prefetched chunks, one warp per CTA
mkdir -p gpurun_out/sr3
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sr3/build.log 2>&1
timeout 900 python -m pytest -q -x tests/test_gpu_scan_slices.py tests/test_gpu_fullsize.py -m gpu -k "scan or cumsum" > gpurun_out/sr3/pytest.log 2>&1; echo pytest rc=$? >> gpurun_out/sr3/pytest.log
for v in "64 1" "32 1" "64 2" "128 1"; do set -- $v
  GRUMPY_SCAN_ROWS_CW=$1 GRUMPY_SCAN_ROWS_WPB=$2 timeout 600 python bench.py --workload cumsum-rows --steps 10 --warmup 3 > gpurun_out/sr3/cw$1_w$2.json 2> gpurun_out/sr3/cw$1_w$2.err
done
