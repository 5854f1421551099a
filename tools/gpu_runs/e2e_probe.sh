mkdir -p gpurun_out/e2e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e2e/build.log 2>&1
for i in 1 2 3; do timeout 300 python tools/e2e_probe.py mlp 25 > gpurun_out/e2e/mlp_$i.txt 2>&1; done
timeout 300 python tools/e2e_probe.py cumsum-rows 15 > gpurun_out/e2e/cr.txt 2>&1
