#!/bin/bash
# Build compile-time variants of libgcx.so into paper_2111_08617_b200/variants/
# (development tool; variants are timed by scripts/variant_bench.py on the GPU).
# usage: scripts/build_variants.sh NAME:"-DFLAG=1 -DFLAG2=0" ...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/paper_2111_08617_b200/variants
CS=$ROOT/paper_2111_08617_b200/csrc
mkdir -p $OUT
rm -f $OUT/*.so
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  ( /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
      -Xcompiler -fPIC -Xptxas -v -I$ROOT/include $flags -shared -o $OUT/$name.so \
      $CS/gcx_kernels.cu $CS/gcx_stats.cu 2> $OUT/$name.ptxas.log \
    && echo "$name: $(grep -A3 'Compiling.*k_quant32' $OUT/$name.ptxas.log | grep -o 'Used [0-9]* registers')" ) &
done
wait
