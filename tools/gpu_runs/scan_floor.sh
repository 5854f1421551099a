# streaming floor of the TMA scan ring (no look-back) against the lag
mkdir -p gpurun_out/sf
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sf/build.log 2>&1
for lag in 1 2 3; do
  GRUMPY_SCAN_LAG=$lag GRUMPY_SCAN_DEFINES=GR_SCAN_NOLB timeout 300 python bench.py --workload cumsum --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/sf/nolb_l$lag.json 2>&1
  GRUMPY_SCAN_LAG=$lag timeout 300 python bench.py --workload cumsum --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 1 > gpurun_out/sf/l$lag.json 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gr_region -s 3 -c 1 -o gpurun_out/sf/full_nolb env GRUMPY_SCAN_DEFINES=GR_SCAN_NOLB python bench.py --workload cumsum --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
