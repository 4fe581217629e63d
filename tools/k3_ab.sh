#!/bin/bash
# K3 A/B on one B200: scorer tests + parity pins with each variant library, K3 SM cycles at HY and C
#   bash tools/k3_ab.sh <out-subdir> "build/ab/lib_x.so ..."
OUT=gpurun_out/${1:-k3ab}; mkdir -p $OUT
for wl in HY C; do bash tools/k3_cycles.sh "" base $wl >> $OUT/cycles.txt 2>&1; done
for lib in $2; do
  DFS_B200_LIB=$lib timeout 900 python -m pytest tests/test_gpu_score_sm100.py tests/test_gpu_parity_pins.py -x -q > $OUT/pytest_$(basename $lib .so).log 2>&1
  echo "$lib pytest rc=$?" >> $OUT/cycles.txt
  for wl in HY C; do bash tools/k3_cycles.sh "$lib" "$(basename $lib .so)" $wl >> $OUT/cycles.txt 2>&1; done
done
for wl in HY C; do bash tools/k3_cycles.sh "" base_end $wl >> $OUT/cycles.txt 2>&1; done
