# scans along the contiguous axis: warp-per-32-lines kernel vs thread-per-line
mkdir -p gpurun_out/sr2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sr2/build.log 2>&1
timeout 900 python -m pytest -q -x tests/test_gpu_scan_slices.py tests/test_gpu_fullsize.py -m gpu -k "scan or cumsum" > gpurun_out/sr2/pytest.log 2>&1; echo pytest rc=$? >> gpurun_out/sr2/pytest.log
for v in "0 64 4" "1 64 4" "1 32 4" "1 128 4" "1 64 8" "1 32 8"; do set -- $v
  GRUMPY_SCAN_ROWS_T=$1 GRUMPY_SCAN_ROWS_CW=$2 GRUMPY_SCAN_ROWS_WPB=$3 timeout 600 python bench.py --workload cumsum-rows --steps 10 --warmup 3 > gpurun_out/sr2/t$1_cw$2_w$3.json 2> gpurun_out/sr2/t$1_cw$2_w$3.err
done
