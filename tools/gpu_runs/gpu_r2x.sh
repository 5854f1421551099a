OUT=gpurun_out/r2x; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python tools/debug_stream_bs.py 2>&1 | tail -20
