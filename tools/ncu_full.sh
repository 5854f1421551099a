#!/bin/bash
# usage: tools/ncu_full.sh WORKLOAD NAME [KERNEL_REGEX] [SKIP]
# one `ncu --set full` capture of a bench workload's kernel -> gpurun_out/NAME.ncu-rep
W=$1; NAME=$2; RX=${3:-gr_region}; SK=${4:-3}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$RX -s $SK -c 1 \
  -o gpurun_out/$NAME python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
  > gpurun_out/$NAME.log 2>&1
echo "ncu $NAME rc=$?"
