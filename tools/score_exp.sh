#!/bin/bash
# K3 isolation experiments: library variants with the softmax, the MMAs and/or the key-tile
# TMA loads compiled out, timed at a config shape (tools/score_bench.py). Run from the repo
# root after `make`; BUILD_ONLY=1 only builds build/ab/libscore_<variant>.so.
set -e
WL=${1:-HY}
OBJS=$(ls build/obj/*.o | grep -v score_sm100)
NVF="-gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -Iinclude -Ipaper_2605_23445_b200/csrc --expt-relaxed-constexpr"
VARIANTS="skip_mma:-DDFS_SCORE_SKIP_MMA skip_softmax:-DDFS_SCORE_SKIP_SOFTMAX skip_tma:-DDFS_SCORE_SKIP_TMA softmax_only:-DDFS_SCORE_SKIP_MMA,-DDFS_SCORE_SKIP_TMA"
mkdir -p build/ab
for vf in $VARIANTS; do
  v=${vf%%:*}; f=${vf#*:}; f=${f//,/ }
  nvcc $NVF $f -c paper_2605_23445_b200/csrc/score_sm100.cu -o build/ab/score_$v.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/ab/libscore_$v.so $OBJS build/ab/score_$v.o -lcudart -lcuda
done
if [ "${BUILD_ONLY:-0}" = "1" ]; then exit 0; fi
python tools/score_bench.py $WL 10 | sed "s/^/full         /"
for vf in $VARIANTS; do
  v=${vf%%:*}
  DFS_B200_LIB=$PWD/build/ab/libscore_$v.so timeout 120 python tools/score_bench.py $WL 10 | sed "s/^/$v /"
done
