OUT=gpurun_out/r3h; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python tools/coop_probe.py base nofold base nofold 2>&1 | tail -5
