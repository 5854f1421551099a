mkdir -p gpurun_out/ec
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ec/build.log 2>&1
for i in 1 2; do
  timeout 300 python bench.py --workload rownorm-y --no-cpu-baseline > gpurun_out/ec/ry_$i.json 2>&1
  timeout 300 python bench.py --workload kmeans --no-cpu-baseline > gpurun_out/ec/km_$i.json 2>&1
done
timeout 300 python tools/e2e_probe.py rownorm-y 15 > gpurun_out/ec/probe_ry.txt 2>&1
