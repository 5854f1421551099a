python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_gemm_boundary.py tests/test_gpu_fullsize.py -x -q -k "skinny or mlp" > gpurun_out/skinny.log 2>&1; echo skinny rc=$?
timeout 600 python bench.py --workload mlp --steps 10 --warmup 3 > gpurun_out/b_mlp.json 2> gpurun_out/b_mlp.err; echo mlp rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/mlp_launches.csv python bench.py --workload mlp --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu rc=$?
tail -n 5 gpurun_out/skinny.log
