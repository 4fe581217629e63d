#!/bin/bash
# Build an A/B variant of the library with a different K2 translation unit (permute.cu):
#   bash tools/k2_variant.sh <label> [nvcc -D flags ...]   -> build/ab/lib_<label>.so
set -e
LBL=$1; shift
OBJS=$(ls build/obj/*.o | grep -v "/permute.o")
NVF="-gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -Iinclude -Ipaper_2605_23445_b200/csrc --expt-relaxed-constexpr"
mkdir -p build/ab
nvcc $NVF "$@" -c paper_2605_23445_b200/csrc/permute.cu -o build/ab/permute_$LBL.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/ab/lib_$LBL.so $OBJS build/ab/permute_$LBL.o -lcudart -lcuda
rm -f build/ab/permute_$LBL.o
echo build/ab/lib_$LBL.so
