# exp2 MUFU/polynomial split sweep (DFS_ATTN_POLY) in K5 SM cycles at HY and C
OUT=gpurun_out/g61; mkdir -p $OUT
for pp in 516 3 38; do DFS_ATTN_POLY=$pp bash tools/k5_cycles.sh "" HY_$pp HY >> $OUT/cycles.txt 2>&1; done
for pp in 38 3 516 2; do DFS_ATTN_POLY=$pp bash tools/k5_cycles.sh "" C_$pp C >> $OUT/cycles.txt 2>&1; done
