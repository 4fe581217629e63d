# K5 A/B in SM cycles (tools/k5_cycles.sh), DRAM bytes, and under the power cap (tools/k5_power.py), HY and C
#   bash tools/k5_ab_power.sh <out-subdir> "build/ab/lib_x.so ..."
OUT=gpurun_out/${1:-k5abp}; mkdir -p $OUT
for lib in "" $2 ""; do
  tag=${lib:-in-tree}
  DFS_B200_LIB=$lib timeout 600 python -m pytest tests/test_gpu_attn_sm100.py -x -q > /dev/null 2>&1; echo "$tag pytest rc=$?" >> $OUT/summary.txt
  for wl in HY C; do
    bash tools/k5_cycles.sh "$lib" "$tag" $wl | grep cycles >> $OUT/summary.txt
    echo "$tag $wl $(DFS_B200_LIB=$lib timeout 300 python tools/k5_power.py $wl 6 2>&1 | tail -1)" >> $OUT/summary.txt
  done
  DFS_B200_LIB=$lib ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct -k regex:attn_sm100 -c 1 --csv python tools/k5_once.py HY 2>/dev/null | grep -E "dram__bytes|hit_rate" | awk -F'","' -v l=$tag '{gsub(/"/,"",$NF); print l, $(NF-2), $NF}' >> $OUT/summary.txt
done
