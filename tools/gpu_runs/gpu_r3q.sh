# k-means: two rows per nearest-centre search
OUT=gpurun_out/r3q; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_reduce.py tests/test_gpu_streaming.py tests/test_gpu_distributed.py -q -x > $OUT/t.log 2>&1; echo tests rc=$?; tail -n 2 $OUT/t.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -k kmeans > $OUT/tf.log 2>&1; echo fullsize rc=$?; tail -n 2 $OUT/tf.log
for pr in 1 0; do for rep in 1 2; do GRUMPY_NEAREST_PAIR=$pr timeout 600 python bench.py --workload kmeans --steps 10 --no-cpu-baseline --e2e-steps 1 > $OUT/km$pr$rep.json 2> $OUT/km$pr$rep.err; echo km pair=$pr $(python -c "
import json; d=json.loads(open('$OUT/km$pr$rep.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['roofline']['compute']['frac'], d['parity']['ok'])" 2>&1 | tail -1); done; done
GRUMPY_DEVICE=0 timeout 600 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 tools/two_rank_check.py > $OUT/two_rank.log 2>&1; echo two_rank rc=$?; tail -2 $OUT/two_rank.log
