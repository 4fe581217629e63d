#!/bin/bash
# usage: bash tools/k5_cycles.sh <library .so or ""> <label> [workload]
# K5 duration in SM cycles (ncu sm__cycles_elapsed.max, serialised launches) at HY: a
# clock-independent A/B measure (CUDA-event timings vary ±2 % with the power-capped clock)
LIB=$1; LBL=$2; WL=${3:-HY}
if [ -n "$LIB" ]; then export DFS_B200_LIB=$LIB; fi
ncu --metrics sm__cycles_elapsed.max,gpu__time_duration.sum --clock-control none -k regex:'attn_(sm100|pp)' -c 3 --csv python tools/k5_once.py $WL 2>/dev/null | grep -E "sm__cycles_elapsed.max|gpu__time" | awk -F'","' -v l=$LBL '{gsub(/"/,"",$NF); print l, $(NF-2), $NF}'
