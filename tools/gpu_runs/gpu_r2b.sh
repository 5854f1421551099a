python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_distributed.py -x -q > gpurun_out/dist.log 2>&1; echo dist rc=$?
for w in rownorm kmeans; do timeout 600 python bench.py --workload $w --gpus 2 --steps 10 --warmup 3 > gpurun_out/b2_$w.json 2> gpurun_out/b2_$w.err; echo b2 $w rc=$?; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo ref rc=$?
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_all.log 2>&1; echo all rc=$?
tail -3 gpurun_out/dist.log gpurun_out/gpu_all.log
