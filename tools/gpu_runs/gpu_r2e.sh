python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
GRUMPY_RANDOM_PROGRAMS=1000 timeout 1500 python -m pytest tests/test_gpu_programs.py -q -x > gpurun_out/random1000.log 2>&1; echo random rc=$?
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/gpu_all.log 2>&1; echo all rc=$?
bash tools/sanitize_all.sh
tail -n 3 gpurun_out/random1000.log gpurun_out/gpu_all.log
