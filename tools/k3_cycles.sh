#!/bin/bash
# usage: bash tools/k5_cycles.sh <library .so or ""> <label> [workload]
# K3 duration in SM cycles (ncu sm__cycles_elapsed.max, serialised launches) at HY: a
# clock-independent A/B measure (CUDA-event timings vary ±2 % with the power-capped clock)
LIB=$1; LBL=$2; WL=${3:-HY}
if [ -n "$LIB" ]; then export DFS_B200_LIB=$LIB; fi
ncu --metrics sm__cycles_elapsed.max,gpu__time_duration.sum --clock-control none -k regex:score_sm100 -c 3 --csv python tools/score_bench.py $WL 2 2>/dev/null | grep -E "sm__cycles_elapsed.max|gpu__time" | awk -F'","' -v l=$LBL '{gsub(/"/,"",$NF); print l, $(NF-2), $NF}'
