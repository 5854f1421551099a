# host NUMA placement vs the e2e (pinned host buffers) numbers
mkdir -p gpurun_out/numa
{
nproc; lscpu | grep -i "numa\|socket\|model name"
BUS=$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | head -1 | tr 'A-F' 'a-f' | sed 's/^00000000/0000/')
echo bus=$BUS; cat /sys/bus/pci/devices/$BUS/numa_node; cat /sys/bus/pci/devices/$BUS/local_cpulist
nvidia-smi topo -m
} > gpurun_out/numa/topo.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/numa/build.log 2>&1
BUS=$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | head -1 | tr 'A-F' 'a-f' | sed 's/^00000000/0000/')
LOCAL=$(cat /sys/bus/pci/devices/$BUS/local_cpulist)
for i in 1 2; do
  timeout 300 python bench.py --workload mlp --no-cpu-baseline > gpurun_out/numa/mlp_free_$i.json 2>&1
  timeout 300 taskset -c $LOCAL python bench.py --workload mlp --no-cpu-baseline > gpurun_out/numa/mlp_local_$i.json 2>&1
  timeout 300 taskset -c $LOCAL python bench.py --workload blackscholes-f32 --no-cpu-baseline > gpurun_out/numa/bs_local_$i.json 2>&1
  timeout 300 python bench.py --workload blackscholes-f32 --no-cpu-baseline > gpurun_out/numa/bs_free_$i.json 2>&1
done
