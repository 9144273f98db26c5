#!/bin/bash
# quick GPU iteration: GPU tests + headline lines of the given configs
#   bash scripts/gpu_check.sh <tag> cfg3 cfg3s_f5 ...
tag=$1; shift
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/$tag.tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/$tag.tests.log
tail -3 gpurun_out/$tag.tests.log
for c in "$@"; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --headline-only > gpurun_out/$tag.$c.json 2>gpurun_out/$tag.$c.err
  python3 -c "
import json,sys; d=json.loads(open('gpurun_out/$tag.$c.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$c', round(d['ms_per_step'],3), 'kernel_ms', round(r['kernel_ms'],3), 'frac', round(r['frac'],4), 'mufu', round(r['mufu_frac'],3), 'evals', r['evaluations'])" || tail -5 gpurun_out/$tag.$c.err
done
