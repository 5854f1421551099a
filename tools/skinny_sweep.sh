#!/bin/bash
# MLP layer-2 skinny prologue configurations: B placement, threads/CTA, rows/thread, stages
for cfg in cbank,64,1,3 cbank,64,2,3 cbank,32,2,4 cbank,32,4,3 smem,64,2,3 smem,128,2,2 smem,128,1,3 smem,64,4,2; do
  GRUMPY_SKINNY_CFG=$cfg timeout 300 python bench.py --workload mlp --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
    > gpurun_out/sk_$cfg.json 2> gpurun_out/sk_$cfg.err
  echo "$cfg rc=$? $(python -c "
import json,sys; d=json.loads(open('gpurun_out/sk_$cfg.json').read().strip().splitlines()[-1]); print(d['parity']['ok'], {k: round(v*1e3,1) for k,v in d['step_breakdown_ms']['per_launch'].items()})" 2>&1 | tail -1)"
done
