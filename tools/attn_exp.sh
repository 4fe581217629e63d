#!/bin/bash
# K5 isolation experiments: build variants of the library with the MMAs or the softmax
# compiled out and time each at HY (tools/attn_bench.py). Run from the repo root.
set -e
OBJS=$(ls build/obj/*.o | grep -v attn_sm100)
NVF="-gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -Iinclude -Ipaper_2605_23445_b200/csrc --expt-relaxed-constexpr"
mkdir -p build/ab
for v in SKIP_MMA SKIP_SOFTMAX SKIP_TMA; do
  nvcc $NVF -DDFS_ATTN_$v -c paper_2605_23445_b200/csrc/attn_sm100.cu -o build/ab/attn_$v.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/ab/lib_$v.so $OBJS build/ab/attn_$v.o -lcudart -lcuda
done
