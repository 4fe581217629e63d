OUT=gpurun_out/g45; mkdir -p $OUT
for pp in 516 84260 70217 102985 67876 74834; do DFS_ATTN_POLY=$pp bash tools/k5_cycles.sh "" HY_poly$pp HY >> $OUT/cycles.txt 2>&1; done
for pp in 516 84260 70217; do DFS_ATTN_POLY=$pp bash tools/k5_cycles.sh "" C_poly$pp C >> $OUT/cycles.txt 2>&1; done
