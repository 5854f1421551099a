OUT=gpurun_out/r3c; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
DUMP=1 timeout 600 python tools/coop_probe.py base rotate rotate_mb2 rotate_mb4 2>&1 | tail -8
