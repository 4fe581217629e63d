OUT=gpurun_out/g26; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_attn_sm100.py -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/summary.txt
bash tools/k5_cycles.sh "" HY_rs_qt HY >> $OUT/cycles.txt 2>&1
bash tools/k5_cycles.sh build/ab/lib_rs_noqt.so HY_rs_noqt HY >> $OUT/cycles.txt 2>&1
bash tools/k5_cycles.sh "" C_rs_qt_p3 C >> $OUT/cycles.txt 2>&1
DFS_ATTN_POLY=38 bash tools/k5_cycles.sh "" C_rs_qt_p38 C >> $OUT/cycles.txt 2>&1
DFS_ATTN_POLY=2 bash tools/k5_cycles.sh "" C_rs_qt_p2 C >> $OUT/cycles.txt 2>&1
bash tools/k5_cycles.sh build/ab/lib_old.so C_old C >> $OUT/cycles.txt 2>&1
bash tools/k5_cycles.sh build/ab/lib_rs_noqt.so C_rs_noqt C >> $OUT/cycles.txt 2>&1
