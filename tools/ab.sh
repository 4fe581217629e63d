#!/bin/bash
# Generic K5 A/B on one B200: for each variant library, the K5 attention tests (parity) and
# K5 SM cycles at HY and C (tools/k5_cycles.sh); the in-tree library first and last (noise).
#   bash tools/ab.sh <out-subdir> "build/ab/lib_x.so build/ab/lib_y.so" [workloads]
OUT=gpurun_out/${1:-ab}; mkdir -p $OUT
WLS=${3:-"HY C"}
for wl in $WLS; do bash tools/k5_cycles.sh "" base $wl >> $OUT/cycles.txt 2>&1; done
for lib in $2; do
  DFS_B200_LIB=$lib timeout 600 python -m pytest tests/test_gpu_attn_sm100.py -x -q > $OUT/pytest_$(basename $lib .so).log 2>&1
  echo "$lib pytest rc=$?" >> $OUT/cycles.txt
  for wl in $WLS; do bash tools/k5_cycles.sh "$lib" "$(basename $lib .so)" $wl >> $OUT/cycles.txt 2>&1; done
done
for wl in $WLS; do bash tools/k5_cycles.sh "" base_end $wl >> $OUT/cycles.txt 2>&1; done
