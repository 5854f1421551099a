# BS f32 with div.full / sqrt.approx in inexact regions; final-fold microbenchmark
OUT=gpurun_out/r3m; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_map.py tests/test_gpu_streaming.py tests/test_gpu_programs.py -q -x > $OUT/t.log 2>&1; echo tests rc=$?; tail -n 2 $OUT/t.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -k blackscholes > $OUT/tf.log 2>&1; echo fullsize rc=$?; tail -n 2 $OUT/tf.log
for fd in 1 0; do GRUMPY_FAST_DIV=$fd timeout 600 python bench.py --steps 20 --no-cpu-baseline --e2e-steps 1 > $OUT/bs$fd.json 2> $OUT/bs$fd.err; echo bs fastdiv=$fd $(python -c "
import json; d=json.loads(open('$OUT/bs$fd.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['roofline']['frac'], d['parity']['ok'], d['parity'].get('max_err'))" 2>&1 | tail -1); done
timeout 600 python bench.py --workload blackscholes-f64 --steps 10 --no-cpu-baseline --e2e-steps 1 > $OUT/bs64.json 2> $OUT/bs64.err; echo bs64 $(python -c "
import json; d=json.loads(open('$OUT/bs64.json').read().strip().splitlines()[-1]); print(d['roofline'].get('kernel_ms'), d['roofline']['frac'], d['parity']['ok'])" 2>&1 | tail -1)
timeout 300 python tools/coop_probe.py fold 2>&1 | tail -2
