#!/bin/bash
# compute-sanitizer over small launches of every hot-path kernel (tools/sanitize.py):
# memcheck and racecheck on the production library, synccheck on the sanitizer build of
# K5 (tools/k5_variant.sh sync ... -DDFS_SYNCCHECK_BUILD), which additionally observes every
# o_done mbarrier phase. Logs -> ${OUT:-gpurun_out/r2}/sanitize_<tool>.log
OUT=${OUT:-gpurun_out/r2}; mkdir -p $OUT
for tool in memcheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py > $OUT/sanitize_$tool.log 2>&1
  echo "sanitize $tool rc=$?"
done
DFS_B200_LIB=build/ab/lib_sync.so timeout 900 compute-sanitizer --tool synccheck --print-limit 20 \
  python tools/sanitize.py > $OUT/sanitize_synccheck.log 2>&1
echo "sanitize synccheck rc=$?"
