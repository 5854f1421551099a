# new defaults (warp tree, one look-back warp, lag 2): scan + streaming + full-size suites, bench, ncu
mkdir -p gpurun_out/tr2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/tr2/build.log 2>&1
timeout 900 python -m pytest -q -x tests/test_gpu_scan_slices.py tests/test_gpu_streaming.py tests/test_gpu_fullsize.py -m gpu > gpurun_out/tr2/pytest.log 2>&1; echo pytest rc=$? >> gpurun_out/tr2/pytest.log
timeout 300 python bench.py --workload cumsum > gpurun_out/tr2/bench_cumsum.json 2> gpurun_out/tr2/bench_cumsum.err
timeout 300 python bench.py --workload cumsum-rows --no-cpu-baseline > gpurun_out/tr2/bench_cumsum-rows.json 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/tr2/launches_cumsum.csv timeout 300 python bench.py --workload cumsum --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gr_region -s 3 -c 1 -o gpurun_out/tr2/full_cumsum timeout 300 python bench.py --workload cumsum --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tr2/scan_rows_probe.csv python tools/scan_rows_probe.py > gpurun_out/tr2/scan_rows_probe.txt 2>&1
