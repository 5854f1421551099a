mkdir -p gpurun_out/sp2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sp2/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sp2/probe.csv python tools/scan_rows_probe.py > gpurun_out/sp2/probe.txt 2>&1
