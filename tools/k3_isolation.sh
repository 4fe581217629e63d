OUT=gpurun_out/k3iso; mkdir -p $OUT
bash tools/k3_cycles.sh "" full HY >> $OUT/cycles.txt 2>&1
for v in skip_mma skip_softmax skip_tma softmax_only; do bash tools/k3_cycles.sh build/ab/libscore_$v.so $v HY >> $OUT/cycles.txt 2>&1; done
