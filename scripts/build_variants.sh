#!/bin/bash
# Build compile-time variants of libgcx.so into paper_2111_08617_b200/variants/
# (development tool; variants are timed by scripts/variant_bench.py on the GPU).
# usage: scripts/build_variants.sh NAME:"-DFLAG=1 -DFLAG2=0" ...
# VARIANT_FILES (default "gcx_span"): the sources rebuilt with the flags; the
# other objects come from the regular build (make -C paper_2111_08617_b200/csrc).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/paper_2111_08617_b200/variants
CS=$ROOT/paper_2111_08617_b200/csrc
FILES=${VARIANT_FILES:-gcx_span}
mkdir -p $OUT
rm -f $OUT/*.so
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v -I$ROOT/include"
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  (
    objs=""
    for f in gcx_kernels gcx_stats gcx_span; do
      if [[ " $FILES " == *" $f "* ]]; then
        $NV $flags -c -o $OUT/$name.$f.o $CS/$f.cu 2>> $OUT/$name.ptxas.log
        objs="$objs $OUT/$name.$f.o"
      else
        objs="$objs $CS/build/$f.cu.o"
      fi
    done
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/$name.so $objs
    rm -f $OUT/$name.*.o
    echo "$name: $(grep -A3 'Compiling.*k_spanILj4ELi7ELb1' $OUT/$name.ptxas.log | grep -o 'Used [0-9]* registers')"
  ) &
done
wait
