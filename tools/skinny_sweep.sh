#!/bin/bash
# MLP layer-2 skinny prologue configurations: B placement, threads/CTA, rows/thread, stages
for cfg in ${CFGS:-smem,128,2,2 l1,64,2,2 l1,64,2,3 l1,32,2,3 l1,64,1,3 l1,128,2,2 l1,32,2,2}; do
  GRUMPY_SKINNY_CFG=$cfg timeout 300 python bench.py --workload mlp --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
    > gpurun_out/sk_$cfg.json 2> gpurun_out/sk_$cfg.err
  echo "$cfg rc=$? $(python -c "
import json,sys; d=json.loads(open('gpurun_out/sk_$cfg.json').read().strip().splitlines()[-1]); print(d['parity']['ok'], {k: round(v*1e3,1) for k,v in d['step_breakdown_ms']['per_launch'].items()})" 2>&1 | tail -1)"
done
