mkdir -p gpurun_out/sr4
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sr4/build.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gr_region -s 3 -c 1 -o gpurun_out/sr4/full_cumsum_rows timeout 600 python bench.py --workload cumsum-rows --steps 1 --warmup 3 > gpurun_out/sr4/ncu.log 2>&1
