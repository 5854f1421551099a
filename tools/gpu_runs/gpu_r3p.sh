# full GPU suite at HEAD + two ranks sharing the GPU + smoke
OUT=gpurun_out/r3p; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/gpu_all.log 2>&1; echo all rc=$?; tail -n 2 $OUT/gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo smoke rc=$?; tail -1 $OUT/smoke.log
GRUMPY_DEVICE=0 timeout 600 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 tools/two_rank_check.py > $OUT/two_rank.log 2>&1; echo two_rank rc=$?; tail -3 $OUT/two_rank.log
