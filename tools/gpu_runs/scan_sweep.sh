# look-back-by-rounds TMA scan: tile size / ring depth / lag sweep (cumsum 2^28)
mkdir -p gpurun_out/ss
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ss/build.log 2>&1
for v in "16 6 2" "16 6 1" "8 12 2" "8 12 3" "8 12 4" "8 10 3" "32 3 1" "16 5 2"; do set -- $v
  GRUMPY_SCAN_TMA=1 GRUMPY_SCAN_ITEMS=$1 GRUMPY_SCAN_STAGES=$2 GRUMPY_SCAN_LAG=$3 timeout 300 python bench.py --workload cumsum --steps 20 --warmup 5 > gpurun_out/ss/i$1_s$2_l$3.json 2>&1
  GRUMPY_SCAN_TMA=1 GRUMPY_SCAN_ITEMS=$1 GRUMPY_SCAN_STAGES=$2 GRUMPY_SCAN_LAG=$3 GRUMPY_SCAN_DEFINES=GR_SCAN_NOLB timeout 300 python bench.py --workload cumsum --steps 20 --warmup 5 > gpurun_out/ss/nolb_i$1_s$2_l$3.json 2>&1
done
