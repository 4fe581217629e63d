#!/bin/bash
# usage (on the GPU box): bash tools/gpu_profile.sh <tag> [workload]
# 1. launch list of the warm-up + profiled update-step calls (cold-cache, serialised: compare shares)
# 2. ncu --set full of the second call's kernels (each launch replayed ~40x)
TAG=${1:-r1}
WL=${2:-HY}
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python tools/profile_step.py $WL > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:'attn_sm100|score_sm100|permute_kernel|topk|absmax|split_kernel|factor_kernel|lut_ptr' -s 12 -c 12 \
  -o gpurun_out/prof_$TAG python tools/profile_step.py $WL > gpurun_out/ncu_$TAG.log 2>&1
ls -la gpurun_out
