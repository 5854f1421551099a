mkdir -p gpurun_out/st
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/st/build.log 2>&1
for lag in 1 2 3; do
GRUMPY_SCAN_TMA=1 GRUMPY_SCAN_LAG=$lag GRUMPY_SCAN_DEFINES=GR_SCAN_STATS timeout 300 python bench.py --workload cumsum --steps 3 --warmup 3 > gpurun_out/st/stats_l$lag.txt 2>&1
done
