#!/bin/bash
# ncu --set full capture of one gbs_fp32_kernel launch (after the 3 warm-up steps):
#   bash scripts/gpu_ncu.sh <config> <out-name> [extra bench args]
c=$1; o=$2; shift 2
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gbs_fp32_kernel -s 3 -c 1 \
  -o gpurun_out/$o python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --headline-only "$@" > gpurun_out/$o.log 2>&1
echo "ncu $c rc=$?" >> gpurun_out/$o.log
