# compute-sanitizer synccheck on K5 sanitizer builds (tools/k5_variant.sh <label> ... -DDFS_SYNCCHECK_BUILD),
# plus the production library's SM cycles for the same change: bash tools/synccheck_ab.sh "sync ..." [prod lib]
mkdir -p gpurun_out/sc
for l in ${1:-sync}; do DFS_B200_LIB=build/ab/lib_$l.so timeout 900 compute-sanitizer --tool synccheck --print-limit 5 python tools/sanitize.py > gpurun_out/sc/$l.log 2>&1; echo "$l rc=$?" >> gpurun_out/sc/summary.txt; done
if [ -n "$2" ]; then for wl in HY C; do bash tools/k5_cycles.sh "" base $wl >> gpurun_out/sc/cycles.txt; bash tools/k5_cycles.sh "$2" prod $wl >> gpurun_out/sc/cycles.txt; done; fi
