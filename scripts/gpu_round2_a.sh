#!/bin/bash
# round-2 measurement batch A: headline lines of the other shapes + one ncu capture
for c in cfg1 cfg2 cfg3s cfg3s_f5 cfg3s_pb; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --headline-only > gpurun_out/line_$c.json 2>gpurun_out/line_$c.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gbs_fp32_kernel -s 1 -c 1 \
  -o gpurun_out/r2a_cfg3 python bench.py --config cfg3 --steps 1 --warmup 1 --no-cpu-baseline --headline-only > gpurun_out/ncu_cfg3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gbs_fp32_kernel -s 1 -c 1 \
  -o gpurun_out/r2a_f5 python bench.py --config cfg3s_f5 --steps 1 --warmup 1 --no-cpu-baseline --headline-only > gpurun_out/ncu_f5.log 2>&1
ls -la gpurun_out
