#!/bin/bash
# bench line (default), reference arm, launch list, one ncu --set full of the summation kernel
timeout 900 python bench.py > gpurun_out/r2g_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/r2_bench.log
timeout 600 python bench.py --impl reference > gpurun_out/r2g_bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/r2_bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2g_launches_cfg3.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --headline-only > gpurun_out/r2g_launches.log 2>&1
bash scripts/gpu_ncu.sh cfg3 r2g_cfg3
bash scripts/gpu_ncu.sh cfg3s_f5 r2g_f5
