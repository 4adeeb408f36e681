#!/bin/bash
# Build a variant of libamgr_b200.so with extra nvcc flags on one source file
# (development A/B; load it with AMGR_LIB=abtest/lib_<name>.so).
# usage: tools/ab_variant.sh <name> <source.cu> "<extra nvcc flags>"
set -e
name=$1; src=$2; extra=$3
here=$(cd "$(dirname "$0")/.." && pwd)
csrc=$here/paper_2108_02054_b200/csrc
mkdir -p $here/abtest/obj_$name
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC,-O2 -cudart static --expt-relaxed-constexpr"
$NV $extra -c $csrc/$src -o $here/abtest/obj_$name/${src%.cu}.o
objs=""
for o in $csrc/build/*.o; do
  b=$(basename $o)
  if [ "$b" == "${src%.cu}.o" ]; then objs="$objs $here/abtest/obj_$name/$b"; else objs="$objs $o"; fi
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $here/abtest/lib_$name.so $objs -ldl
echo built abtest/lib_$name.so
