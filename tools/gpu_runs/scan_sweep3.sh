mkdir -p gpurun_out/ss3
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ss3/build.log 2>&1
for v in "0 2 3" "20 2 3" "64 2 3" "200 2 3" "20 2 2" "64 1 3"; do set -- $v
  GRUMPY_SCAN_TMA=1 GRUMPY_SCAN_SLEEP=$1 GRUMPY_SCAN_LBW=$2 GRUMPY_SCAN_LAG=$3 timeout 300 python bench.py --workload cumsum --steps 20 --warmup 5 > gpurun_out/ss3/sl$1_w$2_l$3.json 2>&1
done
GRUMPY_SCAN_TMA=1 GRUMPY_SCAN_LBW=1 GRUMPY_SCAN_LAG=3 GRUMPY_SCAN_DEFINES=GR_SCAN_NOLB timeout 300 python bench.py --workload cumsum --steps 20 --warmup 5 > gpurun_out/ss3/nolb_w1_l3.json 2>&1
