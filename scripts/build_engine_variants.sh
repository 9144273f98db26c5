#!/bin/bash
# engine.cu variants of libbf_gbs.so (host-path tuning): bash scripts/build_engine_variants.sh "-DX=1" ...
set -e
cd "$(dirname "$0")/../paper_2501_13382_b200/csrc"
mkdir -p ../_lib/variants
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="$ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
for v in "$@"; do
  name=$(echo "$v" | tr ' =' '_-' | tr -d 'D')
  mkdir -p build/evar_$name
  /usr/local/cuda/bin/nvcc $FL $v -c engine.cu -o build/evar_$name/engine.o
  /usr/local/cuda/bin/nvcc $ARCH -shared -o ../_lib/variants/libbf_gbs_e$name.so build/evar_$name/engine.o build/gbs_fp32.o build/exact_fp64.o build/probe.o build/writers.o build/hostpool.o -Xlinker -lpthread
  echo "built $name"
done
