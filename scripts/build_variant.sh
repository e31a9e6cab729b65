#!/bin/bash
# Build an experimental variant of the library: scripts/build_variant.sh <name> <nvcc defines...>
# -> paper_1111_0627_b200/lib/libocm_b200_<name>.so (select with OCM_LIB=...)
set -e
cd "$(dirname "$0")/../paper_1111_0627_b200"
name=$1; shift
out=build/var_$name; mkdir -p $out lib
ARCH="-gencode arch=compute_100a,code=sm_100a"
for f in solver.cu prep.cu gen_dev.cu; do nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 "$@" -c csrc/$f -o $out/$f.o & done
for f in graph.cpp gen.cpp capi.cpp; do nvcc $ARCH -O3 -std=c++17 -Xcompiler -fPIC,-O3 "$@" -x c++ -c csrc/$f -o $out/$f.o & done
wait
nvcc $ARCH -shared -o lib/libocm_b200_$name.so $out/*.o -lcudart -lpthread
echo lib/libocm_b200_$name.so
