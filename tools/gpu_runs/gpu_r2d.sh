python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in cbank smem; do
GRUMPY_SKINNY_B=$v timeout 600 python bench.py --workload mlp --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_mlp_$v.json 2> gpurun_out/b_mlp_$v.err; echo mlp $v rc=$?
GRUMPY_SKINNY_B=$v timeout 900 python -m pytest tests/test_gpu_gemm_boundary.py -x -q -k "skinny or mlp" > gpurun_out/skinny_$v.log 2>&1; echo test $v rc=$?
done
GRUMPY_SKINNY_B=cbank tools/ncu_full.sh mlp mlp_skinny_cbank
GRUMPY_SKINNY_B=smem tools/ncu_full.sh mlp mlp_skinny_smem
