#!/bin/bash
# usage (on the GPU box): bash tools/gpu_profile.sh <tag>
set -x
TAG=${1:-r1}
mkdir -p gpurun_out
# launch list of one warm step (cold-cache, serialised: compare shares)
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python tools/profile_step.py > /dev/null 2>&1
# full capture of the top kernels of the profiled step (last launch of each)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'attn_sm100|score_sm100|permute_kernel|topk_kernel' -s 0 -c 12 -o gpurun_out/prof_$TAG python tools/profile_step.py > gpurun_out/ncu_$TAG.log 2>&1
ls -la gpurun_out
