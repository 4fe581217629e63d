# exp2 MUFU/polynomial split sweep (DFS_ATTN_POLY) in K5 SM cycles at HY and C
OUT=gpurun_out/${1:-poly}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_attn_sm100.py -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/cycles.txt
for pp in 3 516 38 2; do DFS_ATTN_POLY=$pp bash tools/k5_cycles.sh "" HY_$pp HY >> $OUT/cycles.txt 2>&1; done
for pp in 38 3 516 2; do DFS_ATTN_POLY=$pp bash tools/k5_cycles.sh "" C_$pp C >> $OUT/cycles.txt 2>&1; done
