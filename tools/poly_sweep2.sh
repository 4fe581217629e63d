# exp2 split placement sweep (round 2; the back-placed POLY codes 118-122 and 201 it measured were
# removed from attn_sm100.cu after it, see DESIGN §3 and profiles/r2/poly_placement_sweep.txt)
OUT=gpurun_out/${1:-poly2}; mkdir -p $OUT
export DFS_B200_LIB=build/ab/lib_pext.so
for pp in 3 121 120 122 118 201; do DFS_ATTN_POLY=$pp bash tools/k5_cycles.sh "" HY_$pp HY >> $OUT/cycles.txt 2>&1; done
for pp in 38 121 120 122 118 201; do DFS_ATTN_POLY=$pp bash tools/k5_cycles.sh "" C_$pp C >> $OUT/cycles.txt 2>&1; done
DFS_ATTN_POLY=121 timeout 600 python -m pytest tests/test_gpu_attn_sm100.py -x -q > $OUT/pytest.log 2>&1; echo "pytest121 rc=$?" >> $OUT/cycles.txt
