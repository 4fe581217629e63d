#!/bin/bash
# Build an A/B variant of the library with one translation unit recompiled:
#   bash tools/variant.sh <label> <tu (attn_sm100|permute|score_sm100|...)> <source> [nvcc -D flags ...]
# -> build/ab/lib_<label>.so (travels to the GPU box; select it with DFS_B200_LIB=...).
# Run from the repo root after `make`.
set -e
LBL=$1; TU=$2; SRC=$3; shift 3
OBJS=$(ls build/obj/*.o | grep -v "/$TU.o")
NVF="-gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -Iinclude -Ipaper_2605_23445_b200/csrc --expt-relaxed-constexpr"
mkdir -p build/ab
nvcc $NVF "$@" -c "$SRC" -o build/ab/${TU}_$LBL.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/ab/lib_$LBL.so $OBJS build/ab/${TU}_$LBL.o -lcudart
echo build/ab/lib_$LBL.so
