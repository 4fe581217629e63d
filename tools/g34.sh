OUT=gpurun_out/g34; mkdir -p $OUT
DFS_ATTN_PP=1 timeout 600 python -m pytest tests/test_gpu_attn_sm100.py -x -q > $OUT/pytest_pp.log 2>&1; echo "pp rc=$?" >> $OUT/summary.txt
DFS_ATTN_PP=1 bash tools/k5_cycles.sh "" HY_pp HY >> $OUT/cycles.txt 2>&1
bash tools/k5_cycles.sh "" HY_base HY >> $OUT/cycles.txt 2>&1
DFS_ATTN_PP=1 bash tools/k5_cycles.sh "" C_pp C >> $OUT/cycles.txt 2>&1
bash tools/k5_cycles.sh "" C_base C >> $OUT/cycles.txt 2>&1
