OUT=gpurun_out/g44; mkdir -p $OUT
for pp in 3 30 31 516; do DFS_ATTN_POLY=$pp bash tools/k5_cycles.sh "" HY_poly$pp HY >> $OUT/cycles.txt 2>&1; done
for pp in 3 30 31 516; do DFS_ATTN_POLY=$pp bash tools/k5_cycles.sh "" W4_poly$pp W4 >> $OUT/cycles.txt 2>&1; done
