mkdir -p gpurun_out/rm
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/rm/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rm/probe.csv python tools/rows_mid_probe.py > gpurun_out/rm/probe.txt 2>&1
