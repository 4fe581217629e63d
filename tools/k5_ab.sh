# K5 A/B batch on one B200: attention tests, HY and C SM cycles of the in-tree library and of
# the variant libraries named in $2 (tools/k5_variant.sh), one per-block trace (lib_trace.so).
#   bash tools/k5_ab.sh <out-subdir> "build/ab/lib_x.so build/ab/lib_y.so"
OUT=gpurun_out/${1:-g20}; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_attn_sm100.py -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/summary.txt
bash tools/k5_cycles.sh "" HY HY >> $OUT/cycles.txt 2>&1
bash tools/k5_cycles.sh "" C C >> $OUT/cycles.txt 2>&1
for lib in $2; do bash tools/k5_cycles.sh "$lib" "$lib" HY >> $OUT/cycles.txt 2>&1; done
DFS_B200_LIB=build/ab/lib_trace.so timeout 300 python tools/trace_attn.py > $OUT/trace.txt 2>&1
