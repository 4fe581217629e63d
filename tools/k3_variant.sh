#!/bin/bash
# Build an A/B variant of the library with a different K3 translation unit:
#   bash tools/k3_variant.sh <label> <score_sm100 source> [nvcc -D flags ...]
# -> build/ab/lib_<label>.so (travels to the GPU box; select it with DFS_B200_LIB=...).
# Run from the repo root after `make`.
set -e
LBL=$1; SRC=$2; shift 2
OBJS=$(ls build/obj/*.o | grep -v score_sm100)
NVF="-gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -Iinclude -Ipaper_2605_23445_b200/csrc --expt-relaxed-constexpr"
mkdir -p build/ab
nvcc $NVF "$@" -c "$SRC" -o build/ab/score_$LBL.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/ab/lib_$LBL.so $OBJS build/ab/score_$LBL.o -lcudart
echo build/ab/lib_$LBL.so
