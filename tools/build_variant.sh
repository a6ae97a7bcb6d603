#!/bin/bash
# build a variant of libswiftdec_b200.so with one source recompiled under extra flags
#   tools/build_variant.sh <source.cu> <out.so> <nvcc flags...>
src=$1; out=$2; shift 2
B=paper_2502_18890_b200/build
obj=/tmp/variant_$(basename $src .cu)_$$.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
  -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Iinclude -Ipaper_2502_18890_b200/csrc "$@" -c paper_2502_18890_b200/csrc/$src -o $obj || exit 1
objs=$(ls $B/*.o | grep -v "/$(basename ${EXCLUDE:-$src} .cu).o")
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a $objs $obj -o $out -lcudart && rm $obj
