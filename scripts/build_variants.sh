#!/bin/bash
# Build kernel-configuration variants of libbf_gbs.so (tuning sweeps only):
#   bash scripts/build_variants.sh "-DBF_ROWCAP=64" "-DBF_RANGES=32" ...
set -e
cd "$(dirname "$0")/../paper_2501_13382_b200/csrc"
mkdir -p ../_lib/variants
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="$ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
for v in "$@"; do
  name=$(echo "$v" | tr ' =' '_-' | tr -d 'D')
  mkdir -p build/var_$name
  /usr/local/cuda/bin/nvcc $FL $v -c gbs_fp32.cu -o build/var_$name/gbs_fp32.o -Xptxas -v 2> build/var_$name/ptxas.txt
  /usr/local/cuda/bin/nvcc $ARCH -shared -o ../_lib/variants/libbf_gbs_$name.so build/engine.o build/var_$name/gbs_fp32.o build/exact_fp64.o build/probe.o build/writers.o build/hostpool.o -Xlinker -lpthread
  echo "$name $(grep -A2 ILi1E build/var_$name/ptxas.txt | grep -oE 'Used [0-9]+ registers|[0-9]+ bytes spill stores' | tr '\n' ' ')"
done
