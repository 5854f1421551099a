# streamed e2e: chunk size sweep (host bytes in + out per chunk)
mkdir -p gpurun_out/cs
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/cs/build.log 2>&1
for mb in 32 64 128 256; do
  for w in blackscholes-f32 cumsum rownorm; do
    GRUMPY_STREAM_CHUNK_MB=$mb timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/cs/${w}_$mb.json 2>&1
  done
done
