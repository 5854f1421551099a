mkdir -p gpurun_out/sd
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sd/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/sd/pytest_gpu.log 2>&1; echo pytest rc=$? >> gpurun_out/sd/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/sd/smoke.log 2>&1
timeout 300 python bench.py --workload cumsum --steps 20 --warmup 5 > gpurun_out/sd/bench_cumsum.json 2> gpurun_out/sd/bench_cumsum.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sd/launches_cumsum.csv timeout 300 python bench.py --workload cumsum --steps 2 --warmup 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gr_region -s 3 -c 1 -o gpurun_out/sd/full_cumsum timeout 600 python bench.py --workload cumsum --steps 1 --warmup 3 > gpurun_out/sd/ncu_full.log 2>&1
