mkdir -p gpurun_out/ss2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ss2/build.log 2>&1
for v in "16 6 3" "16 6 4" "12 8 3" "12 8 4" "12 8 5" "8 12 4" "8 12 6" "20 5 2" "16 6 3 GR_SCAN_NOLB" "12 8 4 GR_SCAN_NOLB"; do set -- $v
  GRUMPY_SCAN_TMA=1 GRUMPY_SCAN_LBW=2 GRUMPY_SCAN_ITEMS=$1 GRUMPY_SCAN_STAGES=$2 GRUMPY_SCAN_LAG=$3 GRUMPY_SCAN_DEFINES=$4 timeout 300 python bench.py --workload cumsum --steps 20 --warmup 5 > gpurun_out/ss2/i$1_s$2_l$3_$4.json 2>&1
done
