# K5 isolation in SM cycles (HY and C): the in-tree kernel, its MMA/TMA side alone (softmax
# compiled out, -DDFS_ATTN_SKIP_SOFTMAX) and its softmax side alone (MMAs compiled out,
# -DDFS_ATTN_SKIP_MMA); build the variants first with tools/k5_variant.sh skipsm / skipmma.
OUT=${OUT:-gpurun_out/iso}; mkdir -p $OUT
for wl in HY C; do
  bash tools/k5_cycles.sh "" full_$wl $wl >> $OUT/cycles.txt 2>&1
  bash tools/k5_cycles.sh build/ab/lib_skipsm.so mma_side_$wl $wl >> $OUT/cycles.txt 2>&1
  bash tools/k5_cycles.sh build/ab/lib_skipmma.so softmax_side_$wl $wl >> $OUT/cycles.txt 2>&1
done
