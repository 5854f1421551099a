# row scans (bit-exact): lines per warp x warps per CTA x chunk width
mkdir -p gpurun_out/rw
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/rw/build.log 2>&1
for v in "16 1 64" "8 2 64" "16 2 64" "8 4 64" "16 1 32" "8 1 64" "4 4 128"; do set -- $v
  GRUMPY_SCAN_ROWS_RPW=$1 GRUMPY_SCAN_ROWS_WPB=$2 GRUMPY_SCAN_ROWS_CW=$3 timeout 300 python bench.py --workload cumsum-rows --no-cpu-baseline --e2e-steps 1 > gpurun_out/rw/r$1_w$2_c$3.json 2>&1
done
