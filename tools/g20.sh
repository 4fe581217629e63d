# K5 A/B batch: attention tests, HY/C SM cycles of the in-tree library, one trace
OUT=gpurun_out/${1:-g20}; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_attn_sm100.py -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/summary.txt
bash tools/k5_cycles.sh "" HY HY >> $OUT/cycles.txt 2>&1
bash tools/k5_cycles.sh "" C C >> $OUT/cycles.txt 2>&1
for lib in $2; do bash tools/k5_cycles.sh "$lib" "$lib" HY >> $OUT/cycles.txt 2>&1; done
DFS_B200_LIB=build/ab/lib_trace.so timeout 300 python tools/trace_attn.py > $OUT/trace.txt 2>&1
