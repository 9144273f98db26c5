#!/bin/bash
# time every library variant in _lib/variants (and the product library) on the given configs
#   bash scripts/gpu_variants.sh cfg3 cfg3s ...
for c in "$@"; do
  for so in paper_2501_13382_b200/_lib/libbf_gbs.so paper_2501_13382_b200/_lib/variants/*.so; do
    n=$(basename $so .so)
    BF_GBS_LIB=$PWD/$so timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --headline-only > gpurun_out/var.$n.$c.json 2> gpurun_out/var.$n.$c.err
    r=$(tail -1 gpurun_out/var.$n.$c.json | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['ms_per_step'],2), round(r['kernel_ms'],2), round(r['frac'],4))" 2>&1)
    echo "$c $n $r $(grep -h 'bf hist' gpurun_out/var.$n.$c.err | tail -1)"
  done
done
