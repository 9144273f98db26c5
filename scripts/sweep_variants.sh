#!/bin/bash
# Times bench.py --config ${CFG:-cfg3s} with every library variant in _lib/variants
# (run from the repository root: CFG=cfg3 bash scripts/sweep_variants.sh).
for so in paper_2501_13382_b200/_lib/variants/*.so; do
  n=$(basename $so .so)
  r=$(BF_GBS_LIB=$PWD/$so timeout 300 python bench.py --config ${CFG:-cfg3s} --steps 3 --warmup 3 --no-cpu-baseline --headline-only 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), round(d['roofline']['kernel_ms'],2))" 2>&1)
  echo "$n $r"
done
