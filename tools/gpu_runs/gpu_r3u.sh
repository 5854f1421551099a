OUT=gpurun_out/r3u; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python tools/scan_probe.py "stats:GR_SCAN_STATS" "nolb:GR_SCAN_NOLB" 2>&1 | tail -4
