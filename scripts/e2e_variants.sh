#!/bin/bash
for so in paper_2501_13382_b200/_lib/libbf_gbs.so paper_2501_13382_b200/_lib/variants/*.so; do
  echo "== $(basename $so)"; BF_GBS_LIB=$PWD/$so python scripts/e2e_probe.py ${1:-cfg3} 2>&1 | grep "host step\|device step"
done
