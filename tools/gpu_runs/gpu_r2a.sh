set -x
nproc; free -g | head -2; nvidia-smi --query-gpu=name,memory.total --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/fullsize.log 2>&1; echo fullsize rc=$?
for w in blackscholes-f32 rownorm kmeans; do timeout 600 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/b_$w.json 2> gpurun_out/b_$w.err; echo $w rc=$?; done
timeout 600 python bench.py --workload rownorm --gpus 2 --steps 10 --warmup 3 > gpurun_out/b2_rownorm.json 2> gpurun_out/b2_rownorm.err; echo b2 rc=$?
tail -3 gpurun_out/fullsize.log
