OUT=gpurun_out/g43; mkdir -p $OUT
for pp in 38 3 4 2; do DFS_ATTN_POLY=$pp bash tools/k5_cycles.sh "" HY_poly$pp HY >> $OUT/cycles.txt 2>&1; done
for pp in 38 3 2; do DFS_ATTN_POLY=$pp bash tools/k5_cycles.sh "" C_poly$pp C >> $OUT/cycles.txt 2>&1; done
